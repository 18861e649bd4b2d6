#!/bin/bash
# Full measurement pass: parity tests, bench for the configs, launch list and
# an ncu --set full capture of the hot kernels (hurricane).
set -u
OUT=gpurun_out
timeout 600 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 300 > $OUT/gpu_tests.log 2>&1
echo "tests=$?"; tail -1 $OUT/gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench=$?"
for c in ${CONFIGS:-cesm nyx hacc}; do
  timeout 600 python bench.py --steps 10 --warmup 3 --config $c --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo "bench_$c=$?"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"describe|dq|codebook|chunk|inflate|rq|outlier|init_status|resolve|decode_prep|lut" -c 60 --csv --log-file $OUT/launches.csv python tools/profile_step.py hurricane 2 > /dev/null 2>&1
echo "ncu_launch=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU_KERNELS:-inflate_fast|dq3d_tma|rq3d_block|chunk_pack32|chunk_stats|describe|codebook|decode_prep}" -s 8 -c 8 -o $OUT/prof_full python tools/profile_step.py hurricane 2 > /dev/null 2>&1
echo "ncu_full=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"inflate_fast|dq1d_vec|rq1d_rec|chunk_pack32|describe" -c 5 -o $OUT/prof_hacc python tools/profile_step.py hacc 1 > /dev/null 2>&1
echo "ncu_hacc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"describe|dq|codebook|chunk|inflate|rq|outlier|init_status|resolve|decode_prep|lut|task_bounds" -c 60 --csv --log-file $OUT/launches_hacc.csv python tools/profile_step.py hacc 2 > /dev/null 2>&1
echo "ncu_launch_hacc=$?"

#!/bin/bash
# Round-2 measurement pass: GPU parity tests, the default bench line (large
# config), the other configs, an ncu launch list of two large-config steps and
# an ncu --set full capture of the large config's hot kernels.
set -u
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt
if [ -z "${SKIP_TESTS:-}" ]; then
  timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=15 > $OUT/gpu_tests.log 2>&1
  echo "tests=$?"; tail -3 $OUT/gpu_tests.log
fi
timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench_large.json 2> $OUT/bench_large.err; echo "bench=$?"
for c in ${CONFIGS:-hurricane nyx hacc cesm}; do
  timeout 600 python bench.py --steps 20 --warmup 5 --config $c --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo "bench_$c=$?"
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref=$?"
K='describe|dq|codebook|chunk|inflate|rq|outlier|init_status|resolve|decode_prep|lut|task_bounds|quality'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$K" -c 80 --csv --log-file $OUT/launches_large.csv python tools/profile_step.py large 2 > /dev/null 2>&1
echo "ncu_launch_large=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${NCU_KERNELS:-inflate_fast|dq3d_tma|rq3d_block|chunk_pack32|chunk_stats|describe|codebook|decode_prep}" -c 9 -o $OUT/prof_large python tools/profile_step.py large 1 > /dev/null 2>&1
echo "ncu_full_large=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$K" -c 80 --csv --log-file $OUT/launches_hacc.csv python tools/profile_step.py hacc 2 > /dev/null 2>&1
echo "ncu_launch_hacc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"inflate_fast|dq1d_vec|rq1d_rec|chunk_pack32|chunk_stats|describe" -c 6 -o $OUT/prof_hacc python tools/profile_step.py hacc 1 > /dev/null 2>&1
echo "ncu_full_hacc=$?"
# summaries on the box (the .ncu-rep files are too large to bring back)
for c in large hacc; do
  if [ -f $OUT/prof_$c.ncu-rep ]; then
    python tools/ncu_summary.py $OUT/prof_$c.ncu-rep $c $OUT/ncu_full_$c.txt > /dev/null 2>&1
    for k in inflate_fast chunk_pack32 dq3d_tma rq3d_block dq1d_vec rq1d_rec; do
      python tools/ncu_diverge.py $OUT/prof_$c.ncu-rep $k 25 > $OUT/ncu_lines_${c}_$k.txt 2>/dev/null
    done
    [ -n "${KEEP_REP:-}" ] || rm -f $OUT/prof_$c.ncu-rep
  fi
done
python tools/launches.py $OUT/launches_large.csv > $OUT/launches_large.txt 2>/dev/null
python tools/launches.py $OUT/launches_hacc.csv > $OUT/launches_hacc.txt 2>/dev/null
ls -la $OUT | tail -40

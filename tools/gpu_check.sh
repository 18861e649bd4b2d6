#!/bin/bash
# One GPU round: parity tests, a short bench, and the per-kernel launch list.
set -u
OUT=gpurun_out
timeout 700 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 300 -x -p no:cacheprovider > $OUT/gpu_tests.log 2>&1
echo "tests=$?"; tail -4 $OUT/gpu_tests.log | cut -c1-400
timeout 600 python bench.py --steps 10 --warmup 3 ${BENCH_ARGS:-} > $OUT/bench.json 2> $OUT/bench.err
echo "bench=$?"; cut -c1-1800 $OUT/bench.json; tail -3 $OUT/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"dq|codebook|chunk|inflate|rq|describe|resolve|lut|outlier|init|set_eb" -c 40 --csv --log-file $OUT/launches.csv python tools/profile_step.py ${CFG:-hurricane} 2 > /dev/null 2>&1
echo "ncu=$?"
python tools/launches.py $OUT/launches.csv

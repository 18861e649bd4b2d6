set -u
OUT=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=10 > $OUT/gpu_tests.log 2>&1; echo "tests=$?"; tail -3 $OUT/gpu_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 > $OUT/bench_large.json 2> $OUT/bench_large.err; echo "bench=$?"
timeout 600 python tools/kbench.py hurricane nyx hacc cesm large > $OUT/kbench.json 2> $OUT/kbench.err; echo kb=$?

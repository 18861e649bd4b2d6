#!/bin/bash
# generic-shape row kernels: parity (generic shapes, variants, differential), then shape timings
set -u
OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider -k "Generic or pack" > $OUT/rows_tests.log 2>&1
echo "generic_tests=$?"; tail -3 $OUT/rows_tests.log | cut -c1-400
timeout 900 python -m pytest tests/test_gpu_variants.py -q -x -m gpu -p no:cacheprovider -k "ROWS or NO_BLK or STRIP" > $OUT/rows_var.log 2>&1
echo "variant_tests=$?"; tail -3 $OUT/rows_var.log | cut -c1-400
timeout 600 python tools/kbench_blocks.py > $OUT/shapes.json 2> $OUT/shapes.err
echo "shapes=$?"; cut -c1-330 $OUT/shapes.json; tail -3 $OUT/shapes.err

#!/bin/bash
# quick: generic-shape parity (+ strip / rows variants) and the shapes the row kernels serve
set -u
OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider -k "Generic" > $OUT/rows_tests.log 2>&1
echo "generic_tests=$?"; tail -2 $OUT/rows_tests.log | cut -c1-400
timeout 900 python -m pytest tests/test_gpu_variants.py -q -x -m gpu -p no:cacheprovider -k "STRIP or RQ_ROWS" > $OUT/rows_var.log 2>&1
echo "variant_tests=$?"; tail -2 $OUT/rows_var.log | cut -c1-400
timeout 600 python tools/kbench_blocks.py 512,512,512:16,16,16 512,512,512:2,8,32 8192,8192:32,32 8192,8192:4,64 ${EXTRA:-} > $OUT/shapes.json 2> $OUT/shapes.err
echo "shapes=$?"; python -c "
import json
for l in open('$OUT/shapes.json'):
    d=json.loads(l); k=d['kernels']; print(d['dims'], d['block'], d['gbs'], {a:b for a,b in k.items() if 'strip' in a or 'rows' in a or 'blocks' in a or 'seg' in a})"
tail -3 $OUT/shapes.err

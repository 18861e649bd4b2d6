#!/bin/bash
# decoder iteration: parity subset, diagnostics, per-kernel timings
set -u
OUT=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -q -m gpu -x -p no:cacheprovider > $OUT/dec_tests.log 2>&1
echo "tests=$?"; tail -5 $OUT/dec_tests.log | cut -c1-400
timeout 300 python tools/inflate_diag.py hurricane nyx hacc cesm large > $OUT/dec_diag.log 2>&1; echo diag=$?; cat $OUT/dec_diag.log | tail -6
timeout 600 python tools/kbench.py ${CFGS:-hurricane nyx hacc cesm large} > $OUT/kbench.json 2> $OUT/kbench.err
echo "kbench=$?"; python -c "
import json
for l in open('$OUT/kbench.json'):
    d=json.loads(l); k=d['kernels']; print(d['config'], d['gbs'], 'c', d['compress_ms'], 'd', d['decompress_ms'], 'inflate', k.get('inflate_fast_kernel'), 'seq', k.get('inflate_kernel'))
"; tail -3 $OUT/kbench.err

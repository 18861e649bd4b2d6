#!/bin/bash
# decoder tuning: per-kernel timings (and decoder diagnostics) for several slice targets
set -u
OUT=gpurun_out
if [ -z "${NOTEST:-}" ]; then
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -q -m gpu -x -p no:cacheprovider > $OUT/dec_tests.log 2>&1
echo "tests=$?"; tail -2 $OUT/dec_tests.log | cut -c1-300
fi
for t in ${TARGETS:-44}; do
SDQZ_DEC_TARGET=$t timeout 300 python tools/inflate_diag.py ${CFGS:-hurricane nyx hacc cesm large} 2>&1 | sed "s/^/target $t /" | tail -5
SDQZ_DEC_TARGET=$t timeout 600 python tools/kbench.py ${CFGS:-hurricane nyx hacc cesm large} > $OUT/kbench_$t.json 2> $OUT/kbench.err
python -c "
import json
for l in open('$OUT/kbench_$t.json'):
    d=json.loads(l); k=d['kernels']; print('target $t', d['config'], d['gbs'], 'c', d['compress_ms'], 'd', d['decompress_ms'], 'inflate', k.get('inflate_fast_kernel'), 'seq', k.get('inflate_kernel'))
"
done

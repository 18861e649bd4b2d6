#!/bin/bash
# packer iteration: parity subset + per-kernel timings, new vs old packer
set -u
OUT=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -q -m gpu -x -p no:cacheprovider > $OUT/pack_tests.log 2>&1
echo "tests=$?"; tail -2 $OUT/pack_tests.log | cut -c1-300
for v in new old; do
if [ $v = old ]; then export SDQZ_OLD_PACK=1; fi
timeout 600 python tools/kbench.py ${CFGS:-hurricane nyx hacc cesm large} > $OUT/kbench_pack_$v.json 2> $OUT/kbench.err
python -c "
import json
for l in open('$OUT/kbench_pack_$v.json'):
    d=json.loads(l); k=d['kernels']; print('$v', d['config'], d['gbs'], 'c', d['compress_ms'], 'd', d['decompress_ms'], 'pack', k.get('chunk_pack32_kernel'), 'stats', k.get('chunk_stats_kernel'))
"
done

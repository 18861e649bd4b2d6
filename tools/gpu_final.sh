#!/bin/bash
# final pass: full GPU suite, smoke(), the default bench line, the generic-shape table
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > $OUT/final_tests.log 2>&1
echo "tests=$?"; tail -2 $OUT/final_tests.log | cut -c1-300
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/final_smoke.log 2>&1
echo "smoke=$?"; tail -1 $OUT/final_smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/final_bench.json 2> $OUT/final_bench.err; echo "bench=$?"
python -c "
import json; d=json.loads(open('$OUT/final_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['compress_gbs'], d['decompress_gbs'], d['roofline']['frac'], d['e2e']['value'], d['parity'], d['clocks'])"
timeout 900 python tools/kbench_blocks.py > $OUT/final_shapes.json 2> $OUT/final_shapes.err; echo "shapes=$?"

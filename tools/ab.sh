#!/bin/bash
# A/B of library builds: ab.sh "<configs>" lib1.so lib2.so ...  (bench value + top kernels)
CONFIGS=$1; shift
for c in $CONFIGS; do
  for lib in "$@"; do
    SDQZ_LIB_PATH=$PWD/paper_2007_09625_b200/$lib timeout 300 python bench.py --steps 10 --warmup 3 --config $c --no-cpu-baseline 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', '$lib', round(d['value'],1), 'c', round(d['compress_gbs'],1), 'd', round(d['decompress_gbs'],1), {k: round(v*1e3,1) for k, v in list(d['kernel_ms'].items())[:6]})"
  done
done

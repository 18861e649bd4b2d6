#!/bin/bash
# decoder slice-target sweep (codewords per lane slice) with kbench
for t in ${TARGETS:-48 56 64 72 80}; do
  echo "target=$t"
  SDQZ_DEC_TARGET=$t timeout 600 python tools/kbench.py ${CFGS:-large nyx hurricane hacc cesm} 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('  ', d['config'], d['gbs'], d['kernels'].get('inflate_fast_kernel'))"
done

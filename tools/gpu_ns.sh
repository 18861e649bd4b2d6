#!/bin/bash
# decoder variants: parity with the 6-symbol table forced, full parity + config scale on the default choice, kbench
set -u
OUT=gpurun_out
SDQZ_DEC_NS=6 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -p no:cacheprovider > $OUT/ns6_tests.log 2>&1
echo "ns6_tests=$?"; tail -3 $OUT/ns6_tests.log | cut -c1-300
timeout 900 python tools/kbench.py ${CFGS:-large nyx cesm hurricane hacc} > $OUT/kbench.json 2> $OUT/kbench.err
echo "kbench=$?"; cat $OUT/kbench.json | cut -c1-260
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_config_scale.py -q -x -m gpu -p no:cacheprovider > $OUT/def_tests.log 2>&1
echo "def_tests=$?"; tail -3 $OUT/def_tests.log | cut -c1-300

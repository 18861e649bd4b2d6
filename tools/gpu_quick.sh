#!/bin/bash
# parity tests (decode-heavy subset first) + per-kernel timings of the configs
set -u
OUT=gpurun_out
timeout ${TT:-900} python -m pytest ${TESTS:-tests} -q -m gpu -x -p no:cacheprovider > $OUT/quick_tests.log 2>&1
echo "tests=$?"; tail -15 $OUT/quick_tests.log | cut -c1-600
timeout 900 python tools/kbench.py ${CFGS:-hurricane nyx hacc cesm large} > $OUT/kbench.json 2> $OUT/kbench.err
echo "kbench=$?"; cat $OUT/kbench.json; tail -3 $OUT/kbench.err

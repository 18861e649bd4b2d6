#!/bin/bash
# ncu --set full of one kernel family on given configs:  KREGEX=... CFGS="large hurricane" bash tools/gpu_ncu_kernel.sh
set -u
OUT=gpurun_out
for c in ${CFGS:-large}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX}" -c ${NCOUNT:-1} -o $OUT/k_${TAG:-x}_$c python tools/profile_step.py $c 1 > $OUT/k_${TAG:-x}_$c.log 2>&1
  echo "ncu_$c=$?"
done

#!/bin/bash
# ncu --set full of the decoder on the large and HACC configs (source-level)
set -u
OUT=gpurun_out
for c in ${CFGS:-large hacc}; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${K:-inflate_fast}" -c ${NC:-1} -o $OUT/prof_inflate_$c python tools/profile_step.py $c 1 > $OUT/ncu_$c.log 2>&1
echo "ncu_$c=$?"
done

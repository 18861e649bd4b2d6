#!/bin/bash
# ncu --set full of the generic-shape row kernels on two shapes; summaries on the box
set -u
OUT=gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-rq_rows|dq_rows|rq1d_seg}" -c ${NCOUNT:-3} -o $OUT/rows ${CMD:-python tools/kbench_blocks.py 8192,8192:8,8 512,512,512:4,4,4} > $OUT/rows_ncu.log 2>&1
echo "ncu=$?"; tail -3 $OUT/rows_ncu.log
python tools/ncu_pipes.py $OUT/rows.ncu-rep > $OUT/rows_pipes.txt 2>&1; cat $OUT/rows_pipes.txt | cut -c1-250
for k in $(echo "${KREGEX:-rq_rows|dq_rows}" | tr "|" " "); do python tools/ncu_lines.py $OUT/rows.ncu-rep $k 30 > $OUT/rows_lines_$k.txt 2>&1; done
ncu -i $OUT/rows.ncu-rep --page details --csv > $OUT/rows_details.csv 2>&1
ncu -i $OUT/rows.ncu-rep --page raw --csv > $OUT/rows_raw.csv 2>&1
rm -f $OUT/rows.ncu-rep

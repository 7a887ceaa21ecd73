#!/bin/bash
# One `ncu --set full` capture of a kernel family from tools/kernel_drivers.py (run under gpurun):
#   bash tools/ncu_one.sh <tag> <family> <kernel regex> <launches to skip> <launches to capture>
T=$1; fam=$2; rx=$3; skip=${4:-0}; cnt=${5:-1}
O=gpurun_out/$T; mkdir -p $O
timeout 600 python tools/kernel_drivers.py $fam > $O/drv_$fam.log 2>&1 || { echo "driver $fam failed" >> $O/drv_$fam.log; exit 1; }
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$rx" -s $skip -c $cnt \
    -o $O/ncu_$fam python tools/kernel_drivers.py $fam > $O/ncu_$fam.log 2>&1
ncu -i $O/ncu_$fam.ncu-rep --page raw --csv > $O/ncu_$fam.raw.csv 2>/dev/null
ncu -i $O/ncu_$fam.ncu-rep --page source --print-source cuda,sass --csv > $O/ncu_$fam.source.csv 2>/dev/null
gzip -f $O/ncu_$fam.source.csv
[ $(stat -c %s $O/ncu_$fam.ncu-rep 2>/dev/null || echo 0) -gt 6000000 ] && rm -f $O/ncu_$fam.ncu-rep
exit 0

#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:xnor_wconv -s 3 -c 1 -o $O/prof_wconv python tools/r2/wconv_ablate.py ${1:-0} 0 > $O/ncu_wconv.log 2>&1
ncu -i $O/prof_wconv.ncu-rep --page raw --csv > $O/prof_wconv.raw.csv 2>/dev/null
ncu -i $O/prof_wconv.ncu-rep --page source --csv > $O/prof_wconv.source.csv 2>/dev/null
ncu -i $O/prof_wconv.ncu-rep --page details > $O/prof_wconv.details.txt 2>/dev/null
rm -f $O/prof_wconv.ncu-rep
tail -3 $O/ncu_wconv.log

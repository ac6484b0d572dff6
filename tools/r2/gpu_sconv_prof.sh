#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2
C="python tools/r2/conv_once.py auto 0 dbg=${DBG:-0}"
timeout 300 $C > $O/conv_once.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"xnor_sconv" -s 1 -c 1 -o $O/prof_sconv $C > $O/ncu_sconv.log 2>&1
r=$O/prof_sconv
if [ -f $r.ncu-rep ]; then
  ncu -i $r.ncu-rep --page raw --csv > $r.raw.csv 2>/dev/null
  ncu -i $r.ncu-rep --page details > $r.details.txt 2>/dev/null
  ncu -i $r.ncu-rep --page source --csv > $r.source.csv 2>/dev/null
  rm -f $r.ncu-rep
fi
tail -2 $O/ncu_sconv.log

#!/bin/bash
# ncu --set full of the shifted-window conv with the f32 shortcut stream (layer 1 and layer 2 shapes)
mkdir -p gpurun_out/r2/wprof
O=gpurun_out/r2/wprof
CMD="python tools/r2/wconv_ablate.py 1,3 0"
timeout 300 $CMD > $O/plain.log 2>&1 || exit 1
cat $O/plain.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:xnor_wconv -s 3 -c 1 -o $O/wconv_res_l1 python tools/r2/wconv_ablate.py 1 0 > $O/ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:xnor_wconv -s 3 -c 1 -o $O/wconv_res_l2 python tools/r2/wconv_ablate.py 3 0 > $O/ncu2.log 2>&1
for r in $O/wconv_res_l1 $O/wconv_res_l2; do
  ncu -i $r.ncu-rep --page raw --csv > $r.raw.csv 2>/dev/null
  ncu -i $r.ncu-rep --page details > $r.details.txt 2>/dev/null
  ncu -i $r.ncu-rep --page source --csv > $r.source.csv 2>/dev/null
done
ls -la $O

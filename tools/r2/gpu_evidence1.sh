#!/bin/bash
# round-2 early evidence: ncu pipe counters of the CUDA-core engines (POPC, b1 mma.sync)
# and a full capture of ResNet-18's layer-1 binary conv (64 filters, cp.async route)
mkdir -p gpurun_out/r2
O=gpurun_out/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
E="python tools/r2/engine_once.py 4096 4096 4096 popc bmma"
timeout 300 $E > $O/engine_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"xnor_popc|xnor_bmma" -c 2 -o $O/prof_engines $E > $O/ncu_engines.log 2>&1
NET="python tools/net_steps.py resnet18 1"
timeout 300 $NET > $O/net_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"xnor_umma" -s 38 -c 2 -o $O/prof_layer1 $NET > $O/ncu_layer1.log 2>&1
for r in $O/prof_engines $O/prof_layer1; do
  if [ -f $r.ncu-rep ]; then
    ncu -i $r.ncu-rep --page raw --csv > $r.raw.csv 2>/dev/null
    ncu -i $r.ncu-rep --page details > $r.details.txt 2>/dev/null
    ncu -i $r.ncu-rep --page source --csv > $r.source.csv 2>/dev/null
    rm -f $r.ncu-rep
  fi
done
du -sh gpurun_out
echo done

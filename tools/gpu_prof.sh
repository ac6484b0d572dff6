#!/bin/bash
# ncu captures of the conv step (pack + umma) and a large GEMM
mkdir -p gpurun_out
C1="python tools/prof_one.py conv 0 0 0 1"
C2="python tools/prof_one.py gemm 8192 8192 8192 1"
timeout 300 $C1 > gpurun_out/p1.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"xnor_umma|pack_nchw" -s 2 -c 2 -o gpurun_out/prof_conv $C1 > gpurun_out/ncu1.log 2>&1
timeout 300 $C2 > gpurun_out/p2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"xnor_umma" -s 1 -c 1 -o gpurun_out/prof_gemm8k $C2 > gpurun_out/ncu2.log 2>&1
echo done

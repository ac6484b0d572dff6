#!/bin/bash
# ncu --set full captures for profiles/: the c2 bench step's kernels and an 8192^3 GEMM.
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/prof_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"xnor_umma|pack_nchw" -s 6 -c 2 -o gpurun_out/prof_bench_c2 $CMD > gpurun_out/ncu_full.log 2>&1
G="python tools/prof_one.py gemm 8192 8192 8192 2"
timeout 300 $G > gpurun_out/p2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"xnor_umma" -s 1 -c 1 -o gpurun_out/prof_gemm8k $G > gpurun_out/ncu2.log 2>&1
echo done

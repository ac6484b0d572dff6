#!/bin/bash
# profiles for profiles/: bench launch list + full ncu of the conv step kernels + a large GEMM
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/prof_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
timeout 300 $CMD > gpurun_out/prof_plain2.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"xnor_umma|pack_nchw" -s 2 -c 2 -o gpurun_out/prof_bench_c2 $CMD > gpurun_out/ncu_full.log 2>&1
C2="python tools/prof_one.py gemm 8192 8192 8192 1"
timeout 300 $C2 > gpurun_out/p2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"xnor_umma" -s 1 -c 1 -o gpurun_out/prof_gemm8k $C2 > gpurun_out/ncu2.log 2>&1
echo done

#!/bin/bash
# round-2 final evidence: launch list of the default bench (ResNet-18), ncu --set full of the new kernels
# (stride-2 stem, shifted-window conv in both epilogue modes, cluster split-K GEMM), an 8192^3 GEMM, the C2 step
mkdir -p gpurun_out/r2/ev3
O=gpurun_out/r2/ev3
PROF="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $PROF > $O/bench_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/resnet18_bench_launches.csv $PROF > $O/ncu_launches.log 2>&1
NET="python tools/net_steps.py resnet18 1"
timeout 300 $NET > $O/net_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stem_s2|xnor_wconv" -c 3 -o $O/prof_net $NET > $O/ncu_net.log 2>&1
C1="python bench.py --workload c1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $C1 > $O/c1_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"xnor_splitk|pack_rows" -s 6 -c 2 -o $O/prof_c1 $C1 > $O/ncu_c1.log 2>&1
G="python tools/prof_one.py gemm 8192 8192 8192 2"
timeout 300 $G > $O/g8k.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"xnor_umma" -s 1 -c 1 -o $O/prof_gemm8k $G > $O/ncu_g8k.log 2>&1
C2="python bench.py --workload c2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"xnor_umma|pack_nchw" -s 6 -c 2 -o $O/prof_c2 $C2 > $O/ncu_c2.log 2>&1
for r in $O/prof_net $O/prof_c1 $O/prof_gemm8k $O/prof_c2; do
  if [ -f $r.ncu-rep ]; then
    ncu -i $r.ncu-rep --page raw --csv > $r.raw.csv 2>/dev/null
    ncu -i $r.ncu-rep --page details > $r.details.txt 2>/dev/null
    rm -f $r.ncu-rep
  fi
done
du -sh $O

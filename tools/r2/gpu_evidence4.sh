#!/bin/bash
# round-2 evidence for the pre-expanded engines: launch lists, ncu --set full of the GEMM / conv / expansion
# kernels, bench lines of every workload, reference arm, test log
mkdir -p gpurun_out/r2/ev4
O=gpurun_out/r2/ev4
timeout 1800 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_default.log 2>&1; echo "rc=$?" >> $O/bench_default.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.log 2>&1
rm -f $O/bench_sweep.log
for w in c2 c1 gemm4096 gemm8192 gemm16384 gemm4096k65536 gemm4096_2bit lenet; do
  timeout 400 python bench.py --workload $w --steps 10 --warmup 3 >> $O/bench_sweep.log 2>&1
done
PROF="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $PROF > $O/bench_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/resnet18_bench_launches.csv $PROF > $O/ncu_launches.log 2>&1
G="python bench.py --workload gemm8192 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $G > $O/g8k_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/gemm8192_bench_launches.csv $G > $O/ncu_g8k_l.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"xnor_xp|expand_pm1" -s 4 -c 2 -o $O/prof_gemm8k $G > $O/ncu_g8k.log 2>&1
NET="python tools/net_steps.py resnet18 1"
timeout 300 $NET > $O/net_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"xconv_xp|expand_conv" -s 2 -c 2 -o $O/prof_xconv $NET > $O/ncu_net.log 2>&1
B2="python bench.py --workload gemm4096_2bit --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $B2 > $O/b2_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"xnor_xp|expand_code2" -s 4 -c 2 -o $O/prof_2bit $B2 > $O/ncu_2bit.log 2>&1
for r in $O/prof_gemm8k $O/prof_xconv $O/prof_2bit; do
  if [ -f $r.ncu-rep ]; then
    ncu -i $r.ncu-rep --page raw --csv > $r.raw.csv 2>/dev/null
    ncu -i $r.ncu-rep --page details > $r.details.txt 2>/dev/null
    rm -f $r.ncu-rep
  fi
done
du -sh $O
tail -2 $O/pytest_gpu.log; tail -1 $O/smoke.log

#!/bin/bash
# Round-end evidence: tests, bench (all workloads), engine contest, ncu launch list +
# full captures.  Outputs land in gpurun_out/ (summaries are copied to profiles/ by hand).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
rm -f gpurun_out/bench_sweep.log
for w in c1 gemm4096 gemm8192 gemm16384 gemm4096k65536 gemm4096_2bit lenet resnet18; do
  timeout 400 python bench.py --workload $w --steps 10 --warmup 3 >> gpurun_out/bench_sweep.log 2>&1
done
timeout 600 python tools/engine_contest.py > gpurun_out/contest.md 2>&1
PROF="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $PROF > gpurun_out/prof_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $PROF > gpurun_out/ncu_launches.log 2>&1
echo done

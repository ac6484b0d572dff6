#!/bin/bash
# One GPU session: tests, bench, launch list + ncu full capture of the conv kernel.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
for w in c1 gemm4096 gemm8192 gemm16384 gemm4096k65536; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/bench_sweep.log 2>&1
done
PROF="python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 300 $PROF > gpurun_out/prof_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $PROF > gpurun_out/ncu_launches.log 2>&1
timeout 300 $PROF > gpurun_out/prof_plain2.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:xnor_umma -s 1 -c 1 -o gpurun_out/prof_umma_c2 $PROF > gpurun_out/ncu_full.log 2>&1
echo done

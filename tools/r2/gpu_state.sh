#!/bin/bash
# state check after a container restore: full GPU tests, smoke, default bench, sweep, launch list
mkdir -p gpurun_out/r2
O=gpurun_out/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 2400 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_default.log 2>&1; echo "rc=$?" >> $O/bench_default.log
rm -f $O/bench_sweep.log
for w in c2 c1 gemm8192 gemm16384 gemm4096_2bit lenet; do
  timeout 400 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline >> $O/bench_sweep.log 2>&1
done
PROF="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_resnet.csv $PROF > $O/ncu_launches.log 2>&1
tail -3 $O/pytest_gpu.log; tail -2 $O/smoke.log; tail -2 $O/bench_default.log
grep '^{' $O/bench_sweep.log | cut -c1-300

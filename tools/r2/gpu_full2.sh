#!/bin/bash
# full GPU test suite, smoke, default bench, sweep, launch list
mkdir -p gpurun_out/r2
O=gpurun_out/r2
timeout 2400 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log; tail -1 $O/smoke.log
timeout 600 python bench.py > $O/bench_default.log 2>&1; echo "rc=$?" >> $O/bench_default.log
tail -2 $O/bench_default.log | cut -c1-700
rm -f $O/bench_sweep.log
for w in c2 c1 gemm8192 lenet; do
  timeout 400 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline >> $O/bench_sweep.log 2>&1
done
grep '^{' $O/bench_sweep.log | cut -c1-260
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.log 2>&1; tail -1 $O/bench_reference.log | cut -c1-400
PROF="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/resnet18_bench_launches.csv $PROF > $O/ncu_launches.log 2>&1

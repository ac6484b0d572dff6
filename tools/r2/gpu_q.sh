#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2
timeout 2400 python -m pytest -q -x -m gpu tests > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --steps 30 > $O/q_bench.log 2>&1
tail -1 $O/q_bench.log | cut -c1-300
timeout 600 python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-300

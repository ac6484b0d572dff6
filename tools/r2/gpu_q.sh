#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_nets.py tests/test_gpu_signpack.py > $O/q_tests.log 2>&1; echo "rc=$?" >> $O/q_tests.log
tail -2 $O/q_tests.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 30 > $O/q_bench.log 2>&1
tail -1 $O/q_bench.log | cut -c1-200
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 30 > $O/q_bench2.log 2>&1
tail -1 $O/q_bench2.log | cut -c1-200

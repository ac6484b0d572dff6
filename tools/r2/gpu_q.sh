#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2
timeout 2400 python -m pytest -q -m gpu tests > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
for i in 1 2 3; do timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_nets.py tests/test_multi_rank_cuda.py 2>&1 | tail -1; done

#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_nets.py tests/test_multi_rank_cuda.py 2>&1 | tail -2
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 30 2>/dev/null | tail -1 | cut -c60-120; done

#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2
timeout 1500 python -m pytest -q -x -m gpu tests/test_gpu_parity.py -k "bitplane or 2bit or planes" > $O/xp_tests.log 2>&1; echo "rc=$?" >> $O/xp_tests.log
tail -15 $O/xp_tests.log
timeout 600 python bench.py --workload gemm4096_2bit --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-600

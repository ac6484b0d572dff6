#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_parity.py tests/test_gpu_signpack.py -k "gemm40 or sweep504 or tail_and_layout or large_gemm or bitplane or pre_expanded" 2>&1 | tail -2
timeout 300 python tools/r2/xp_check.py time 4096x4096x4096 8192x8192x8192 16384x16384x16384 4096x4096x65536 | grep xp
G="python bench.py --workload gemm8192 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $G > $O/g8k_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/g8k_launches.csv $G > /dev/null 2>&1
grep -E "expand_pm1|xnor_xp" $O/g8k_launches.csv | tail -4 | cut -d, -f5,15- | cut -c1-60,200-

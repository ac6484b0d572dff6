#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2
timeout 1500 python -m pytest -q -x -m gpu tests/test_gpu_parity.py -k "gemm40 or sweep504 or tail_and_layout or large_gemm" > $O/xp_tests.log 2>&1; echo "rc=$?" >> $O/xp_tests.log
tail -4 $O/xp_tests.log
for w in gemm4096 gemm8192 gemm16384 gemm4096k65536; do
timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-1500
done > $O/xp_bench.log
cat $O/xp_bench.log

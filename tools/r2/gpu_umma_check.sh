#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_signpack.py -q -m gpu -x > $O/umma_tests.log 2>&1; echo "rc=$?" >> $O/umma_tests.log
tail -3 $O/umma_tests.log
for w in gemm8192 gemm4096 c2 gemm4096k65536; do
  timeout 400 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read())
print(d['config']['workload'][:50], round(d['value'],1), d['unit'], 'step ms', round(d['ms_per_step'],4), 'kernel ms', round(d['roofline']['kernel_ms'],4), 'frac', round(d['roofline']['frac'],3))
"
done

#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > $O/pytest_parity.log 2>&1; echo "rc=$?" >> $O/pytest_parity.log; tail -2 $O/pytest_parity.log
for w in c2 c1 gemm4096 gemm8192 gemm16384 gemm4096k65536; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bw_$w.log 2>&1
  python -c "
import json,sys
for l in open('$O/bw_$w.log'):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print('$w', round(d['value'],1), d['unit'], 'ms', round(d['ms_per_step'],4), 'kern_ms', round(r['kernel_ms'],4), 'frac', round(r['frac'],3))
"
done

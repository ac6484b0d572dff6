#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2
timeout 1800 python -m pytest tests/test_gpu_signpack.py tests/test_gpu_nets.py tests/test_gpu_parity.py -q -m gpu -x > $O/l3_tests.log 2>&1; echo "rc=$?" >> $O/l3_tests.log; tail -3 $O/l3_tests.log
for w in resnet18 c2; do timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read())
print(d['config']['workload'][:40], round(d['value'],1), 'ms', round(d['ms_per_step'],4), 'kernel', round(d['roofline']['kernel_ms'],4), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],1))
"; done

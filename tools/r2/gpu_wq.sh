#!/bin/bash
# quick check of the shifted-window conv: parity tests, then timing with / without the pipelined shortcut stream
mkdir -p gpurun_out/r2
O=gpurun_out/r2
timeout 900 python -m pytest -q -x tests/test_gpu_signpack.py tests/test_gpu_nets.py > $O/wq_test.log 2>&1; echo "rc=$?" >> $O/wq_test.log
tail -4 $O/wq_test.log
timeout 300 python tools/r2/wconv_ablate.py 0,1,2,3,11,12 0 64 2>&1 | tail -20

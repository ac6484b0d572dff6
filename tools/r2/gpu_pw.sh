#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2
timeout 900 python -m pytest -q -x tests/test_gpu_signpack.py -k "pointwise" > $O/pw_test.log 2>&1; echo "rc=$?" >> $O/pw_test.log
tail -15 $O/pw_test.log
timeout 300 python tools/r2/pw_time.py 2>&1 | tail -12

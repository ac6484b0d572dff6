#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2
timeout 600 python -m pytest -q -x -m gpu tests/test_gpu_signpack.py -k "pre_expanded" > $O/xconv_tests.log 2>&1; echo "rc=$?" >> $O/xconv_tests.log
tail -30 $O/xconv_tests.log

#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2
for v in P; do
  BNN_LIB_PATH=$PWD/build/variants/lib$v.so timeout 300 python -m pytest -q -x tests/test_gpu_signpack.py -s -k "small_channel and plain" > $O/bisect_$v.log 2>&1; echo "rc=$?" >> $O/bisect_$v.log
  tail -2 $O/bisect_$v.log
done

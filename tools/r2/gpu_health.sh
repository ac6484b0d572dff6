#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2
nvidia-smi > $O/health_smi.txt 2>&1
timeout 300 python -m pytest -q -x tests/test_gpu_signpack.py -k "conv_sign_pack and not small" > $O/health_old.log 2>&1; echo "rc=$?" >> $O/health_old.log; tail -2 $O/health_old.log
BNN_LIB_PATH=$PWD/build/variants/libP.so CUDA_LAUNCH_BLOCKING=1 timeout 300 python -m pytest -q -x tests/test_gpu_signpack.py -k "small_channel and plain" > $O/health_P.log 2>&1; echo "rc=$?" >> $O/health_P.log; tail -2 $O/health_P.log
grep -n "Error\|error" $O/health_P.log | head -5

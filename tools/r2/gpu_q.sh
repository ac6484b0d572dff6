#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2
timeout 2400 python -m pytest -q -m gpu tests > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
tail -2 $O/pytest_gpu.log
timeout 600 python tools/r2/shard_times.py 2>&1 | grep resnet

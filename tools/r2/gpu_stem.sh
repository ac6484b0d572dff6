#!/bin/bash
# stride-2 stem kernel (bnn_stem_s2.cu): accuracy / bit-identity tests, then timing against the old kernel
mkdir -p gpurun_out/r2
O=gpurun_out/r2
timeout 600 python -m pytest tests/test_gpu_nets.py -q -m gpu -x -k "stem or conv2d_f32 or resnet" > $O/stem_tests.log 2>&1; echo "rc=$?" >> $O/stem_tests.log
tail -15 $O/stem_tests.log
timeout 300 python tools/stem_bench.py 256 > $O/stem_bench_new.log 2>&1; cat $O/stem_bench_new.log
BNN_STEM_OLD=1 timeout 300 python tools/stem_bench.py 256 > $O/stem_bench_old.log 2>&1; cat $O/stem_bench_old.log

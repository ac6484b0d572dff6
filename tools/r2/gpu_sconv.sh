#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2
timeout 600 python -m pytest -q -x tests/test_gpu_signpack.py -k small_channel > $O/sconv_test.log 2>&1; echo "rc=$?" >> $O/sconv_test.log
tail -5 $O/sconv_test.log
if grep -q "rc=0" $O/sconv_test.log; then
  timeout 900 python -m pytest -q -x tests/test_gpu_nets.py tests/test_gpu_signpack.py > $O/sconv_nets.log 2>&1; echo "rc=$?" >> $O/sconv_nets.log
  tail -3 $O/sconv_nets.log
  timeout 300 python tools/layer_bench.py > $O/layer_bench.txt 2>&1
  timeout 600 python bench.py --no-cpu-baseline --steps 20 > $O/bench_resnet_sconv.log 2>&1
  tail -c 2500 $O/bench_resnet_sconv.log
fi

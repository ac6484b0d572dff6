#!/bin/bash
# quick: new GPU tests + the default bench + N>1 code paths (gloo ranks sharing the GPU)
mkdir -p gpurun_out/r2
O=gpurun_out/r2
timeout 900 python -m pytest -q tests/test_multi_rank_cuda.py tests/test_gpu_nets.py tests/test_modelio.py tests/test_cli.py tests/test_integration_stub.py > $O/pytest_new.log 2>&1; echo "rc=$?" >> $O/pytest_new.log
timeout 600 python bench.py > $O/bench_default.log 2>&1; echo "rc=$?" >> $O/bench_default.log
timeout 600 python bench.py --workload c2 --no-cpu-baseline > $O/bench_c2.log 2>&1; echo "rc=$?" >> $O/bench_c2.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.log 2>&1; echo "rc=$?" >> $O/bench_ref.log
for w in resnet18 gemm4096 gemm4096_2bit c2; do
  timeout 600 python bench.py --gpus 2 --backend gloo --workload $w --steps 5 --warmup 3 > $O/bench_g2_$w.log 2>&1; echo "rc=$?" >> $O/bench_g2_$w.log
done
tail -2 $O/*.log

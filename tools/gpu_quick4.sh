mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/layer_bench.py 256 64 56 56 64 3 1 1 > gpurun_out/layer_bench.txt 2>&1
timeout 300 python bench.py --workload resnet18 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_resnet.log 2>&1

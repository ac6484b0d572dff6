mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1
timeout 300 python bench.py --workload gemm8192 --steps 10 --warmup 3 --no-cpu-baseline >> gpurun_out/bench.log 2>&1
timeout 300 python bench.py --workload resnet18 --steps 10 --warmup 3 --no-cpu-baseline >> gpurun_out/bench.log 2>&1
timeout 300 python tools/layer_bench.py > gpurun_out/layer_bench.txt 2>&1

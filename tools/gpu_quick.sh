# quick GPU loop: new tests first, then the full gpu suite, then benches
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_signpack.py tests/test_gpu_nets.py -x -q > gpurun_out/pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_new.log
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/layer_bench.py > gpurun_out/layer_bench.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1
timeout 300 python bench.py --workload resnet18 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_resnet.log 2>&1
timeout 300 python bench.py --workload lenet --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_lenet.log 2>&1
timeout 300 python tools/profile_net.py resnet18 > gpurun_out/prof_resnet.txt 2>&1
echo done

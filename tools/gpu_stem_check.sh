mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_nets.py -x -q -k "stem or resnet" > gpurun_out/pytest_stem.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_stem.log
timeout 300 python bench.py --workload resnet18 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_resnet.log 2>&1
timeout 300 python tools/profile_net.py resnet18 > gpurun_out/prof_resnet.txt 2>&1

mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_nets.py -x -q > gpurun_out/pytest_stem.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_stem.log
python tools/stem_bench.py > gpurun_out/stem_bench.txt 2>&1
timeout 300 python bench.py --workload resnet18 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_resnet.log 2>&1
timeout 300 python bench.py --workload lenet --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_lenet.log 2>&1
python tools/profile_net.py lenet > gpurun_out/prof_lenet.txt 2>&1

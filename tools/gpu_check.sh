mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 400 python bench.py --workload resnet18 --steps 10 --warmup 3 > gpurun_out/bench_resnet.log 2>&1
timeout 300 python tools/profile_net.py resnet18 > gpurun_out/prof_resnet.txt 2>&1
timeout 300 python tools/profile_net.py lenet > gpurun_out/prof_lenet.txt 2>&1
echo done

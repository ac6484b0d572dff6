timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3 >> gpurun_out/exp_pd.log
timeout 300 python bench.py --steps 20 --warmup 3 2>&1 | tail -1 >> gpurun_out/exp_pd.log
for w in gemm4096 gemm8192 gemm4096k65536 c1 resnet18; do timeout 300 python bench.py --workload $w --steps 10 --warmup 3 2>&1 | tail -1 | cut -c1-200 >> gpurun_out/exp_pd.log; done

timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "run_host or pack_rows or pack_cases or qfc or config1" 2>&1 | tail -3 > gpurun_out/exp_pd.log
timeout 300 python bench.py --steps 20 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_c2.json
timeout 300 python bench.py --workload c1 --steps 20 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_c1.json

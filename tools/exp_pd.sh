timeout 300 python bench.py --steps 20 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_c2.json
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2 > gpurun_out/exp_pd.log

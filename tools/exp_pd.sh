timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2 > gpurun_out/exp_pd.log
timeout 300 python tools/race_check.py 5 >> gpurun_out/exp_pd.log 2>&1
for d in 0 1027; do BNN_UMMA_DEBUG=$d timeout 60 python tools/umma_dbg.py 4096 4096 4096 >> gpurun_out/exp_pd.log 2>&1; done
BNN_UMMA_DEBUG=16 timeout 60 python tools/umma_stages.py 4096 4096 4096 > gpurun_out/stages.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_c2.json

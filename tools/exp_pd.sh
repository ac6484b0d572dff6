timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3 > gpurun_out/exp_pd.log
timeout 300 python tools/race_check.py 3 2>&1 | grep v2 >> gpurun_out/exp_pd.log
for d in 0 4096; do for w in c2 c1 gemm4096 gemm8192; do echo "dbg $d $w $(BNN_UMMA_DEBUG=$d timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms'])")" >> gpurun_out/exp_pd.log; done; done

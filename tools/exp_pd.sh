timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2 > gpurun_out/exp_pd.log
timeout 300 python tools/race_check.py 3 2>&1 | grep v2 >> gpurun_out/exp_pd.log
for w in c2 c1 gemm4096; do echo "$w $(timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['pack_ms_est'])")" >> gpurun_out/exp_pd.log; done

timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2 > gpurun_out/exp_pd.log
timeout 300 python tools/profile_net.py resnet18 2>&1 | grep -E "bn_relu|implicit|xnor|pack" | cut -c1-60,150-175 >> gpurun_out/exp_pd.log
echo "resnet $(timeout 300 python bench.py --workload resnet18 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])")" >> gpurun_out/exp_pd.log

mkdir -p gpurun_out; rm -f gpurun_out/pack_sweep.txt
for ch in 8 16 32; do
  echo "CH=$ch" >> gpurun_out/pack_sweep.txt
  for r in 1 2; do
  BNN_PACK_CH=$ch timeout 120 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | python -c "import sys,json; [print(round(json.loads(l)['value'],1), round(json.loads(l)['ms_per_step']*1e3,2), round(json.loads(l)['roofline']['pack_ms_est']*1e3,2)) for l in sys.stdin if l.startswith('{')]" >> gpurun_out/pack_sweep.txt
  done
done

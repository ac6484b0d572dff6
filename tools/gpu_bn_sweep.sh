mkdir -p gpurun_out
rm -f gpurun_out/bn_sweep.txt
for bn in 0 96 128 160 176 192 224 352 384; do
  echo "BN=$bn" >> gpurun_out/bn_sweep.txt
  BNN_FP4_BN=$bn timeout 120 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | python -c "import sys,json; [print(round(json.loads(l)['value'],1), round(json.loads(l)['roofline']['kernel_ms']*1e3,2)) for l in sys.stdin if l.startswith('{')]" >> gpurun_out/bn_sweep.txt
done

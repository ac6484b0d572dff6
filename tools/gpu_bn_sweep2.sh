mkdir -p gpurun_out
rm -f gpurun_out/bn_sweep2.txt
for w in gemm8192 gemm4096; do
for bn in 0 160 176 192 208 224; do
  echo "$w BN=$bn" >> gpurun_out/bn_sweep2.txt
  BNN_FP4_BN=$bn timeout 120 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | python -c "import sys,json; [print(round(json.loads(l)['value'],1), round(json.loads(l)['roofline']['kernel_ms']*1e3,2)) for l in sys.stdin if l.startswith('{')]" >> gpurun_out/bn_sweep2.txt
done
done

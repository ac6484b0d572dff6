# layer1-shape conv (C64 F64 56x56, batch 256) under engine variants / debug ablations
S="256 64 56 56 64 3 1 1 256 128 28 28 128 3 1 1"
for v in 1 0; do
  echo "variant $v"; BNN_UMMA_VARIANT=$v python tools/layer_bench.py $S
done
echo "skip epilogue (2048)"; BNN_UMMA_DEBUG=2048 python tools/layer_bench.py $S
echo "skip f32 stores (1024)"; BNN_UMMA_DEBUG=1024 python tools/layer_bench.py $S
echo "no PDL (65536)"; BNN_UMMA_DEBUG=65536 python tools/layer_bench.py $S

#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2
timeout 600 python bench.py > $O/bench_default.log 2>&1; echo "rc=$?" >> $O/bench_default.log
tail -2 $O/bench_default.log | cut -c1-1500
for n in c2 resnet18; do timeout 300 python tools/r2/e2e_chunks.py $n 2 4 8 16 32 2>&1 | tail -6; done

#!/bin/bash
# Round-end evidence: tests, bench (all workloads), engine contest, ncu launch lists and
# full captures.  Outputs land in gpurun_out/ (summaries are copied to profiles/ by hand).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
rm -f gpurun_out/bench_sweep.log
for w in c1 gemm4096 gemm8192 gemm16384 gemm4096k65536 gemm4096_2bit lenet resnet18; do
  timeout 400 python bench.py --workload $w --steps 10 --warmup 3 >> gpurun_out/bench_sweep.log 2>&1
done
timeout 600 python tools/engine_contest.py > gpurun_out/contest.md 2>&1
timeout 300 python tools/layer_bench.py > gpurun_out/layer_bench.txt 2>&1
timeout 300 python tools/stem_bench.py > gpurun_out/stem_bench.txt 2>&1
PROF="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $PROF > gpurun_out/prof_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $PROF > gpurun_out/ncu_launches.log 2>&1
NET="python tools/net_steps.py resnet18 2"
timeout 300 $NET > gpurun_out/net_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/resnet_launches.csv $NET > gpurun_out/ncu_net.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"xnor_umma|pack_nchw" -s 6 -c 2 -o gpurun_out/prof_bench_c2 $PROF > gpurun_out/ncu_full.log 2>&1
G="python tools/prof_one.py gemm 8192 8192 8192 2"
timeout 300 $G > gpurun_out/p2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"xnor_umma" -s 1 -c 1 -o gpurun_out/prof_gemm8k $G > gpurun_out/ncu2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"conv_pool_kernel" -s 1 -c 1 -o gpurun_out/prof_stem python tools/stem_bench.py > gpurun_out/ncu3.log 2>&1
# keep gpurun_out/ under the copy-back limit: raw-page CSVs instead of the reports
for r in gpurun_out/prof_bench_c2 gpurun_out/prof_gemm8k gpurun_out/prof_stem; do
  if [ -f $r.ncu-rep ]; then
    ncu -i $r.ncu-rep --page raw --csv > $r.raw.csv 2>/dev/null
    ncu -i $r.ncu-rep --page details > $r.details.txt 2>/dev/null
    rm -f $r.ncu-rep
  fi
done
du -sh gpurun_out
echo done

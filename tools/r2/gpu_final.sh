#!/bin/bash
# end-of-round evidence at HEAD: tests, smoke, default bench, sweep, reference arm, launch list,
# per-launch DRAM bytes of one ResNet-18 step, ncu --set full of the new / changed kernels
mkdir -p gpurun_out/r2/final
O=gpurun_out/r2/final
timeout 2400 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log; tail -1 $O/smoke.log
timeout 600 python bench.py > $O/bench_default.log 2>&1; echo "rc=$?" >> $O/bench_default.log
tail -2 $O/bench_default.log | cut -c1-300
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.log 2>&1
rm -f $O/bench_sweep.log
for w in c2 c1 gemm4096 gemm8192 gemm16384 gemm4096k65536 gemm4096_2bit lenet; do
  timeout 400 python bench.py --workload $w --steps 10 --warmup 3 >> $O/bench_sweep.log 2>&1
done
grep '^{' $O/bench_sweep.log | cut -c1-200
PROF="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $PROF > $O/bench_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/resnet18_bench_launches.csv $PROF > $O/ncu_launches.log 2>&1
NET="python tools/net_steps.py resnet18 1"
timeout 300 $NET > $O/net_plain.log 2>&1 && \
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file $O/resnet18_dram_per_launch.csv $NET > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"xnor_pw|xnor_wconv" -c 12 -o $O/prof_l12 $NET > $O/ncu_l12.log 2>&1
for r in $O/prof_l12; do
  if [ -f $r.ncu-rep ]; then
    ncu -i $r.ncu-rep --page raw --csv > $r.raw.csv 2>/dev/null
    ncu -i $r.ncu-rep --page details > $r.details.txt 2>/dev/null
    rm -f $r.ncu-rep
  fi
done
timeout 300 python tools/r2/pw_time.py > $O/pw_time.txt 2>&1
timeout 300 python tools/r2/write_bw.py > $O/write_bw.txt 2>&1
timeout 300 python tools/r2/wconv_ablate.py 0,1,2,3 0 > $O/wconv_times.txt 2>&1
du -sh $O

#!/bin/bash
# round-2 evidence: ncu pipe counters of every engine (POPC, b1 mma.sync, tcgen05 mxf4) at 4096^3,
# full captures of the ResNet-18 stem, the layer-1 small-channel conv, the C2 conv and an 8192^3 GEMM,
# and compute-sanitizer memcheck / racecheck of smoke()
mkdir -p gpurun_out/r2/ev2
O=gpurun_out/r2/ev2
E="python tools/r2/engine_once.py 4096 4096 4096 popc bmma umma2"
timeout 300 $E > $O/engine_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"xnor_popc|xnor_bmma|xnor_umma" -c 3 -o $O/prof_engines $E > $O/ncu_engines.log 2>&1
NET="python tools/net_steps.py resnet18 1"
timeout 300 $NET > $O/net_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"conv_pool_kernel|xnor_sconv" -c 3 -o $O/prof_net $NET > $O/ncu_net.log 2>&1
G="python tools/prof_one.py gemm 8192 8192 8192 2"
timeout 300 $G > $O/g8k.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"xnor_umma" -s 1 -c 1 -o $O/prof_gemm8k $G > $O/ncu_g8k.log 2>&1
PROF="python bench.py --workload c2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"xnor_umma|pack_nchw" -s 6 -c 2 -o $O/prof_c2 $PROF > $O/ncu_c2.log 2>&1
timeout 900 compute-sanitizer --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" > $O/memcheck_smoke.log 2>&1; echo "rc=$?" >> $O/memcheck_smoke.log
timeout 900 compute-sanitizer --tool racecheck python -c "import __graft_entry__ as g; g.smoke()" > $O/racecheck_smoke.log 2>&1; echo "rc=$?" >> $O/racecheck_smoke.log
timeout 900 compute-sanitizer --tool synccheck python -c "import __graft_entry__ as g; g.smoke()" > $O/synccheck_smoke.log 2>&1; echo "rc=$?" >> $O/synccheck_smoke.log
for r in $O/prof_engines $O/prof_net $O/prof_gemm8k $O/prof_c2; do
  if [ -f $r.ncu-rep ]; then
    ncu -i $r.ncu-rep --page raw --csv > $r.raw.csv 2>/dev/null
    ncu -i $r.ncu-rep --page details > $r.details.txt 2>/dev/null
    ncu -i $r.ncu-rep --page source --csv > $r.source.csv 2>/dev/null
    rm -f $r.ncu-rep
  fi
done
du -sh gpurun_out
tail -3 $O/*.log

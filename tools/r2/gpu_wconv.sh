#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2
timeout 900 python -m pytest -q -x tests/test_gpu_signpack.py -k small_channel > $O/wconv_test.log 2>&1; echo "rc=$?" >> $O/wconv_test.log
tail -5 $O/wconv_test.log
if grep -q "rc=0" $O/wconv_test.log; then
  timeout 900 python -m pytest -q -x tests/test_gpu_nets.py tests/test_gpu_signpack.py > $O/wconv_nets.log 2>&1; echo "rc=$?" >> $O/wconv_nets.log
  tail -3 $O/wconv_nets.log
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 20 > $O/bench_resnet_wconv.log 2>&1
  tail -1 $O/bench_resnet_wconv.log | cut -c1-400
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/wconv_launches.csv python tools/net_steps.py resnet18 1 > /dev/null 2>&1
  python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/r2/wconv_launches.csv')))
i=next(i for i,r in enumerate(rows) if 'Kernel Name' in r)
d=rows[i+1:]
for r in d[-34:]:
    print(r[4][:100], r[8], r[-1])
PY
fi

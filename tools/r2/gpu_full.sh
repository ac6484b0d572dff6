#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2
timeout 2400 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --steps 20 > $O/bench_resnet.log 2>&1; echo "rc=$?" >> $O/bench_resnet.log
python - <<'PY'
import json
l = open("gpurun_out/r2/bench_resnet.log").read().strip().splitlines()
for x in l:
    if x.startswith("{"):
        d = json.loads(x)
        print("value", d["value"], "ms", d["ms_per_step"], "e2e", d["e2e"]["value"])
        for k, v in d["roofline"]["families"].items():
            print("  ", k, round(v["ms"], 3), v["launches"])
PY

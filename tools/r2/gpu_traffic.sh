#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_stemroof.log 2>&1; tail -1 $O/bench_stemroof.log | python -c "
import sys, json
d = json.loads(sys.stdin.read())
print(d['value'], d['ms_per_step'], d['e2e']['value'])
print(json.dumps(d['roofline']['stem']))
"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file $O/resnet18_dram_per_launch.csv python tools/net_steps.py resnet18 1 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.reader(open('gpurun_out/r2/resnet18_dram_per_launch.csv')))
i = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[i]; d = rows[i + 1:]
ci = {n: j for j, n in enumerate(h)}
by = collections.OrderedDict()
for r in d:
    by.setdefault(r[ci['ID']], {'name': r[ci['Kernel Name']]})[r[ci['Metric Name']]] = float(r[ci['Metric Value']]); by[r[ci['ID']]]['unit_' + r[ci['Metric Name']]] = r[ci['Metric Unit']]
ids = list(by)
# last step = launches after the last stem kernel
last = max(k for k, i_ in enumerate(ids) if 'stem' in by[i_]['name'])
tot = 0.0
for i_ in ids[last:]:
    e = by[i_]
    def b(m):
        v = e.get(m, 0.0); u = e.get('unit_' + m, 'byte')
        return v * {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}.get(u, 1)
    rd, wr = b('dram__bytes_read.sum'), b('dram__bytes_write.sum')
    fam = 'xnor_' in e['name']
    if fam: tot += rd + wr
    print(f"{e['name'][:70]:70s} read {rd/1e6:9.2f} MB write {wr/1e6:9.2f} MB time {e.get('gpu__time_duration.sum', 0):10.0f}")
print('binary conv family DRAM bytes per step:', tot)
PY

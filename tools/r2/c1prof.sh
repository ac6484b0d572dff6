timeout 400 python bench.py --workload c1 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read())
print(d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline'].get('pack_ms_est'))
"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --workload c1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep -E "splitk|xnor_umma|pack_rows" | tail -8 | cut -c1-220

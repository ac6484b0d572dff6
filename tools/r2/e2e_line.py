"""stdin: one bench.py JSON line -> workload, device value, e2e value / ms, slice count."""
import json
import sys

d = json.loads(sys.stdin.read())
p = d["e2e"]["path"]
i = p.find("pipelined over")
print(d["config"]["workload"][:44], "| value", round(d["value"], 1), "| e2e", round(d["e2e"]["value"], 1),
      "|", round(d["e2e"]["ms_per_step"], 4), "ms |", p[i:i + 32] if i >= 0 else "")

"""Key metrics of `ncu --set full` captures (the `--page raw --csv` export) -> JSON.

    python tools/ncu_summary.py out.json name1=file1.raw.csv name2=file2.raw.csv ...

One entry per profiled launch: duration, DRAM bytes, tensor / ALU / shared-memory pipe
utilisation, issue activity, achieved occupancy, registers, grid -- the numbers DESIGN.md
and bench.py's roofline object quote."""
import csv
import json
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor.sum",
    "sm__inst_executed_pipe_alu.sum",
    "sm__inst_executed_pipe_xu.sum",
    "sm__inst_executed_pipe_lsu.sum",
    "sm__inst_executed_pipe_uniform.sum",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.avg.per_cycle_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "sm__cycles_elapsed.max",
    "sm__cycles_elapsed.avg.per_second",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
]


def summarize(path):
    rows = list(csv.reader(open(path, newline="")))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    names, units = rows[hdr], rows[hdr + 1]
    out = []
    for r in rows[hdr + 2:]:
        if len(r) != len(names):
            continue
        d = dict(zip(names, r))
        u = dict(zip(names, units))
        e = {"kernel": d["Kernel Name"][:160]}
        for k in KEYS:
            if k in d and d[k] != "":
                e[k] = f"{d[k]} {u[k]}".strip()
        # every pipe-instruction counter the capture holds (the engine contest: POPC runs on the
        # ALU / integer pipes, the b1 mma.sync emulation and tcgen05 on the tensor pipe)
        for k in d:
            if k.startswith("sm__inst_executed_pipe_") and k.endswith(".sum") and d[k] not in ("", "0") and k not in e:
                e[k] = f"{d[k]} {u[k]}".strip()
        out.append(e)
    return out


if __name__ == "__main__":
    res = {}
    for a in sys.argv[2:]:
        name, path = a.split("=", 1)
        res[name] = summarize(path)
    json.dump(res, open(sys.argv[1], "w"), indent=1)
    for name, lst in res.items():
        for e in lst:
            print(name, "::", e["kernel"][:90], e.get("gpu__time_duration.sum"),
                  "tensor%", e.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
                  "dram%", e.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"))

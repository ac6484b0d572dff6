#!/usr/bin/env python
"""Benchmark of the B200 binarise -> bit-pack -> xnor-popcount hot path.

Default workload = BASELINE.json configs[1]: QConvolution 3x3, 256 -> 256
filters, input 32x256x28x28 f32 ~ N(0,1), stride 1, pad 1 (GEMM view M=256,
N=32*28*28=25088, K=2304).  A step = sign+pack of the f32 activations
resident in HBM + the implicit-im2col xnor conv writing f32 NCHW output.
Metric: binary TOPS = 2*M*N*K / step time (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload c2|c1|gemm4096|gemm8192|gemm16384|gemm4096k65536]

N > 1 runs under torchrun: every rank runs its own replica of the batch
(weak scaling, no collective on the data path); time = max over ranks.
``--impl reference`` times the reference's CPU algorithm (the pinned oracle
port, oracle/, all host threads) on the same workload; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

METRIC = "xnor-popcount binary TOPS (2MNK/s)"
UNIT = "TOPS"
# arithmetic type of the tcgen05 engine: 1-bit operands expanded in SMEM to e2m1
# (kind::mxf4; the 2-bit planes and cp.async-fed shapes use u8 / kind::i8), exact
# integer counts accumulated in f32 / s32
DTYPE = "b1 -> e2m1 x e2m1 (tcgen05 kind::mxf4), exact f32 counts"
WORKLOADS = ("c2", "c1", "gemm4096", "gemm8192", "gemm16384", "gemm4096k65536", "gemm4096_2bit",
             "lenet", "resnet18")
NET_WORKLOADS = {"lenet": ("binary LeNet (BASELINE configs[2]) images/s", 1024, (1, 28, 28)),
                 "resnet18": ("binary ResNet-18 (BASELINE configs[3]) images/s", 256, (3, 224, 224))}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=30)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=("b200", "reference"), default="b200")
    p.add_argument("--workload", choices=WORKLOADS, default="c2")
    p.add_argument("--algo", default="auto")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    return p.parse_args()


# ----------------------------------------------------------------- workloads
def workload_desc(name):
    import workloads as wl
    if name in NET_WORKLOADS:
        desc, batch, chw = NET_WORKLOADS[name]
        return dict(workload=desc + f", batch {batch} per GPU, input {chw} "
                    + ("U[0,1]" if name == "lenet" else "N(0,1)") + ", random-init weights",
                    M=0, N=0, K=0, batch=batch, seed=3 if name == "lenet" else 4)
    if name == "c2":
        c = wl.C2
        oh = (c["h"] + 2 * c["pad"][0] - c["kh"]) // c["stride"][0] + 1
        ow = (c["w"] + 2 * c["pad"][1] - c["kw"]) // c["stride"][1] + 1
        return dict(workload="QConvolution3x3 256->256, x 32x256x28x28 f32, stride 1 pad 1 "
                    "(BASELINE configs[1])", M=c["f"], N=c["b"] * oh * ow,
                    K=c["c"] * c["kh"] * c["kw"], batch=c["b"], seed=c["seed"])
    if name == "c1":
        c = wl.C1
        return dict(workload="QFullyConnected 4096->1024, batch 256 (BASELINE configs[0])",
                    M=c["units"], N=c["batch"], K=c["k"], batch=c["batch"], seed=c["seed"])
    sizes = {"gemm4096": (4096,) * 3, "gemm8192": (8192,) * 3, "gemm16384": (16384,) * 3,
             "gemm4096k65536": (4096, 4096, 65536), "gemm4096_2bit": (4096,) * 3}
    m, n, k = sizes[name]
    if name.endswith("_2bit"):
        return dict(workload=f"2-bit GEMM (act_bit=weight_bit=2, quantize() of U[0,1]) M={m} "
                    f"N={n} K={k} (BASELINE configs[4]); TOPS = logical 2MNK/s",
                    M=m, N=n, K=k, batch=n, seed=m + n + k + 2)
    return dict(workload=f"binary GEMM M={m} N={n} K={k} (BASELINE configs[4])", M=m, N=n, K=k,
                batch=n, seed=m + n + k)


def build_plan(name, algo):
    import torch

    import workloads as wl
    import paper_1705_09864_b200 as bnn
    from paper_1705_09864_b200.plan import ConvPlan, DensePlan, GemmPlan

    if name == "c2":
        c = wl.C2
        x, w = wl.config2_inputs()
        layer = bnn.QConvolution(c["c"], c["f"], (c["kh"], c["kw"]), c["stride"], c["pad"])
        layer.weight = w
        layer.pack()
        layer.algo = algo
        plan = ConvPlan(layer, c["b"], c["h"], c["w"])
        host_x = torch.from_numpy(x).pin_memory()
        plan.x.copy_(host_x)
        return plan, host_x
    if name == "c1":
        a, w = wl.config1_inputs()
        layer = bnn.QFullyConnected(a.shape[1], w.shape[0], domain="dot")
        layer.weight = w
        layer.pack()
        layer.algo = algo
        plan = DensePlan(layer, a.shape[0])
        host_x = torch.from_numpy(a).pin_memory()
        plan.x.copy_(host_x)
        return plan, host_x
    d = workload_desc(name)
    if name in NET_WORKLOADS:
        from paper_1705_09864_b200 import nets
        from paper_1705_09864_b200.plan import NetPlan
        _, batch, chw = NET_WORKLOADS[name]
        net = nets.lenet_c3(d["seed"]) if name == "lenet" else nets.resnet18_c4(d["seed"])
        net.pack_for_inference()
        g = torch.Generator(device="cuda").manual_seed(d["seed"])
        plan = NetPlan(net, batch, chw)
        if name == "lenet":
            plan.x.copy_(torch.rand(plan.x.shape, device="cuda", generator=g))
        else:
            plan.x.copy_(torch.randn(plan.x.shape, device="cuda", generator=g))
        return plan, plan.x.cpu().pin_memory()
    if name.endswith("_2bit"):
        from paper_1705_09864_b200.bitpack import pack_planes_device
        from paper_1705_09864_b200.plan import BitplanePlan
        g = torch.Generator(device="cuda").manual_seed(d["seed"])
        wf = torch.rand((d["M"], d["K"]), device="cuda", generator=g)
        xf = torch.rand((d["N"], d["K"]), device="cuda", generator=g)
        ap = pack_planes_device(wf, 2, "unsigned")
        bp = pack_planes_device(xf, 2, "unsigned")
        return BitplanePlan(ap, bp, d["K"]), bp.cpu().pin_memory()
    g = torch.Generator(device="cuda").manual_seed(d["seed"])
    W = (d["K"] + 63) // 64
    aw = torch.randint(-2**63, 2**63 - 1, (d["M"], W), device="cuda", generator=g).view(torch.uint64)
    bw = torch.randint(-2**63, 2**63 - 1, (d["N"], W), device="cuda", generator=g).view(torch.uint64)
    plan = GemmPlan(aw, bw, d["K"], algo=algo)
    return plan, bw.cpu().pin_memory()


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi-equivalent sampling through NVML while the timed region runs."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, device_index):
        self.samples, self.reasons = [], 0
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": [n for b, n in self.REASONS.items() if self.reasons & b],
                "samples": len(self.samples)}


# ----------------------------------------------------------------- CPU path
def cpu_reference_step(name, sample_frac_hint=None):
    """One step of the reference algorithm on the host (oracle port, all threads).

    Returns (seconds, binary_ops_done, sample_description).
    """
    from oracle import oracle as orc
    import workloads as wl

    threads = os.cpu_count() or 1
    if name == "c2":
        c = wl.C2
        x, w = wl.config2_inputs()
        nb = sample_frac_hint or c["b"]
        xs = np.ascontiguousarray(x[:nb])
        t0 = time.perf_counter()
        y = orc.qconv_packed(xs, w, c["stride"], c["pad"], threads)
        dt = time.perf_counter() - t0
        d = workload_desc(name)
        ops = 2 * d["M"] * (d["N"] * nb // c["b"]) * d["K"]
        return dt, ops, f"{nb} of {c['b']} images: im2col+binarize+pack_matrix_b+xnor_gemm", y
    if name == "c1":
        a, w = wl.config1_inputs()
        t0 = time.perf_counter()
        y = orc.qfc_dot(a, w, threads)
        dt = time.perf_counter() - t0
        d = workload_desc(name)
        return dt, 2 * d["M"] * d["N"] * d["K"], "full batch: binarize+pack+xnor_gemm", y
    d = workload_desc(name)
    if name in NET_WORKLOADS:
        import torch
        from oracle import nets_ref
        from paper_1705_09864_b200 import nets
        _, batch, chw = NET_WORKLOADS[name]
        nb = sample_frac_hint or 1
        net = _CPU_NETS.get(name)
        if net is None:
            net = nets.lenet_c3(d["seed"]) if name == "lenet" else nets.resnet18_c4(d["seed"])
            _CPU_NETS[name] = net
        rng = np.random.default_rng(d["seed"])
        x = (rng.random((nb,) + chw, dtype=np.float32) if name == "lenet"
             else rng.standard_normal((nb,) + chw, dtype=np.float32))
        t0 = time.perf_counter()
        y = nets_ref.forward(net, x, threads)
        dt = time.perf_counter() - t0
        return dt, nb, f"{nb} of {batch} images: full forward, reference layer semantics", y
    if name.endswith("_2bit"):
        # the reference's only multi-bit path: float BLAS on quantized values
        # (QDense(bits=2) INFER_FLOAT, layers.py:370-377)
        rows = sample_frac_hint or min(d["M"], 256)
        rng = np.random.default_rng(d["seed"])
        wq = orc.quantize(rng.random((rows, d["K"]), dtype=np.float32), 2).astype(np.float32)
        xq = orc.quantize(rng.random((d["N"], d["K"]), dtype=np.float32), 2).astype(np.float32)
        t0 = time.perf_counter()
        y = xq @ wq.T
        dt = time.perf_counter() - t0
        return dt, 2 * rows * d["N"] * d["K"], f"{rows} of {d['M']} rows: f32 BLAS on quantize() values", y
    rows = sample_frac_hint or min(d["M"], 256)
    rng = np.random.default_rng(d["seed"])
    W = (d["K"] + 63) // 64
    aw = rng.integers(0, 2**63, size=(rows, W), dtype=np.uint64)
    bw = rng.integers(0, 2**63, size=(W, d["N"]), dtype=np.uint64)
    t0 = time.perf_counter()
    y = orc.xnor_gemm(aw, bw, threads)
    dt = time.perf_counter() - t0
    return dt, 2 * rows * d["N"] * d["K"], f"{rows} of {d['M']} rows: xnor_gemm_parallel", y


_CPU_NETS = {}


def calibrate_cpu_sample(name, budget_s=2.0):
    """Pick a sample size whose single step takes about budget_s."""
    import workloads as wl
    if name == "c1":
        return None
    if name in NET_WORKLOADS:
        dt, _, _, _ = cpu_reference_step(name, 1)
        return int(max(1, min(NET_WORKLOADS[name][1], budget_s / max(dt, 1e-3))))
    if name == "c2":
        dt, _, _, _ = cpu_reference_step(name, 1)
        return int(max(1, min(wl.C2["b"], budget_s / max(dt, 1e-3))))
    d = workload_desc(name)
    dt, _, _, _ = cpu_reference_step(name, 16)
    return int(max(16, min(d["M"], 16 * budget_s / max(dt, 1e-3))))


def cpu_baseline(name, seconds=12.0):
    sample = calibrate_cpu_sample(name)
    times, ops, desc = [], 0, ""
    t_end = time.perf_counter() + seconds
    while True:
        dt, ops, desc, _ = cpu_reference_step(name, sample)
        times.append(dt)
        if time.perf_counter() > t_end and len(times) >= 3:
            break
    med = statistics.median(times)
    if name in NET_WORKLOADS:
        return {"value": ops / med, "unit": "images/s", "cores": os.cpu_count(), "kind": "port",
                "sample": f"{desc}; median of {len(times)} runs ({med * 1e3:.1f} ms each)",
                "seconds_per_step": med}
    return {"value": ops / med / 1e12, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
            "sample": f"{desc}; median of {len(times)} runs ({med * 1e3:.1f} ms each)",
            "seconds_per_step": med}


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    name = args.workload
    sample = calibrate_cpu_sample(name)
    for _ in range(args.warmup):
        cpu_reference_step(name, sample)
    times, ops, desc = [], 0, ""
    for _ in range(args.steps):
        dt, ops, desc, _ = cpu_reference_step(name, sample)
        times.append(dt)
    total = sum(times)
    is_net = name in NET_WORKLOADS
    value = ops * len(times) / total / (1.0 if is_net else 1e12)
    metric = NET_WORKLOADS[name][0] if is_net else METRIC
    unit = "images/s" if is_net else UNIT
    d = workload_desc(name)
    line = {
        "impl": "reference", "metric": metric, "value": value, "unit": unit, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / len(times) * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (seeded, BASELINE.json shapes)",
        "config": {"workload": d["workload"], "M": d["M"], "N": d["N"], "K": d["K"],
                   "parallelism": "host threads"},
        "cpu_baseline": {"value": value, "unit": unit, "cores": os.cpu_count(), "kind": "port",
                         "sample": desc},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU arm
def load_traffic(name, algo):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        t = json.load(open(p))
        return t.get(f"{name}:{algo}") or t.get(name)
    except Exception:
        return None


def popc_peak_tops():
    """Measured POPC issue rate x 64 binary ops (bnn_probe_pipe_peak)."""
    import ctypes

    import torch
    from paper_1705_09864_b200 import _lib
    lib = _lib.load()
    sink = torch.zeros(1, dtype=torch.int32, device="cuda")
    rate = ctypes.c_double(0)
    _lib.check(lib.bnn_probe_pipe_peak(0, 4096, sink.data_ptr(), ctypes.byref(rate),
                                       _lib.stream_ptr()), "probe")
    return rate.value * 64 / 1e12


def int8_tensor_peak_tops(n=8192, reps=10):
    """Measured dense int8 tensor-core rate: cuBLASLt via torch._int_mm, best of reps."""
    import torch
    a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
    for _ in range(3):
        torch._int_mm(a, b)
    best = float("inf")
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch._int_mm(a, b)
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    del a, b
    return 2 * n ** 3 / (best * 1e-3) / 1e12


def tcgen05_peak_tops(kind):
    """Measured dense tcgen05.mma issue rate (bnn_probe_pipe_peak pipe 1 = kind::i8,
    2 = kind::mxf4) as binary TOPS: 2 x MAC/s (one binary op pair per MAC)."""
    import ctypes

    import torch
    from paper_1705_09864_b200 import _lib
    lib = _lib.load()
    sink = torch.zeros(1, dtype=torch.int32, device="cuda")
    rate = ctypes.c_double(0)
    _lib.check(lib.bnn_probe_pipe_peak(1 if kind == "i8" else 2, 4096, sink.data_ptr(),
                                       ctypes.byref(rate), _lib.stream_ptr()), "probe")
    return 2 * rate.value / 1e12


def pipe_peak(algo, workload="c2"):
    """Roofline denominator for the engine that ran (all measured on this GPU)."""
    popc = popc_peak_tops()
    if algo in ("auto", "umma"):
        # TMA-fed shapes run the kind::mxf4 engine (variant 2); the 2-bit planes run kind::i8
        kind = "i8" if workload.endswith("2bit") else "mxf4"
        return {"bound": "tensor", "peak": tcgen05_peak_tops(kind), "unit": "TOPS",
                "peak_source": f"measured: dense tcgen05.mma kind::{kind} issue rate, one CTA per "
                               "SM, 128x256 MMAs back to back (bnn_probe_pipe_peak); the engine "
                               f"runs kind::{kind} on bits expanded in SMEM",
                "popc_peak": popc, "cublas_int8_tops": int8_tensor_peak_tops()}
    return {"bound": "popc", "peak": popc, "unit": "TOPS",
            "peak_source": "measured: bnn_probe_pipe_peak POPC rate x 64 binary ops "
                           "(32 bits x {xor, add})", "popc_peak": popc}


def run_gpu_arm(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local_rank)
    import paper_1705_09864_b200 as bnn
    bnn.load_library()

    plan, host_x = build_plan(args.workload, args.algo)
    d = workload_desc(args.workload)
    ops = plan.binary_ops
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MiB > L2
    flush_rd = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    flush_sink = torch.empty((), dtype=torch.float32, device="cuda")

    def l2_flush():
        # write a buffer larger than L2 (evicts every line of this step's data), then
        # read another one so the dirty lines of the write are written back here, outside
        # the timed region, instead of inside the next timed kernel (a steady-state L2
        # holds clean data, not 126 MB of dirty scratch)
        flush.zero_()
        torch.amax(flush_rd, dim=0, out=flush_sink)
    stream = torch.cuda.current_stream()

    # Each step is replayed from a CUDA graph (pack + kernel) so the events time
    # GPU work only; the kernel alone is a second graph, timed the same way,
    # for the roofline.  Capture happens on a side stream (torch requirement).
    g_step, g_kern = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(stream)
    with torch.cuda.stream(side):
        plan.run_device()
    torch.cuda.synchronize()
    with torch.cuda.graph(g_step):
        plan.run_device()
    with torch.cuda.graph(g_kern):
        plan.kernel()
    for _ in range(args.warmup):
        g_step.replay()
    torch.cuda.synchronize()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    evk = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        for i in range(args.steps):
            l2_flush()  # L2 flush between timed steps (outside the events)
            s, e = ev[i]
            s.record(stream)
            g_step.replay()
            e.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    for i in range(args.steps):  # kernel alone, same flush discipline
        l2_flush()
        s, e = evk[i]
        s.record(stream)
        g_kern.replay()
        e.record(stream)
    torch.cuda.synchronize()
    step_ms = [s.elapsed_time(e) for s, e in ev]
    kern_ms = [s.elapsed_time(e) for s, e in evk]
    pack_ms = [max(0.0, a - b) for a, b in zip(step_ms, kern_ms)]
    total_ms = sum(step_ms)
    plan.check_flags()
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    is_net = args.workload in NET_WORKLOADS
    units_per_step = d["batch"] if is_net else ops / 1e12  # images or tera-ops
    metric = NET_WORKLOADS[args.workload][0] if is_net else METRIC
    unit = "images/s" if is_net else UNIT
    value = world * units_per_step / (ms_per_step * 1e-3)

    # end to end through the public plan API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        y_host = torch.empty(plan.y.shape, dtype=plan.y.dtype).pin_memory()
        for _ in range(2):
            plan.run_host(host_x, y_host)
        if world > 1:
            dist.barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0.record(stream)
        for _ in range(args.steps):
            plan.run_host(host_x, y_host)
        t1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = t0.elapsed_time(t1)
        if world > 1:
            t = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": world * units_per_step / (e2e_ms / args.steps * 1e-3), "unit": unit,
               "h2d_bytes_per_step": plan.h2d_bytes, "d2h_bytes_per_step": plan.d2h_bytes,
               "ms_per_step": e2e_ms / args.steps,
               "path": "plan.run_host: pinned H2D -> pack -> kernel -> D2H -> sync (one CUDA-graph "
                       "replay per call, pipelined over "
                       f"{getattr(plan, 'host_chunks', 1)} batch slices on 3 streams)"}

    peak = pipe_peak(args.algo, args.workload)
    kern_avg = statistics.mean(kern_ms)
    achieved = ops / (kern_avg * 1e-3) / 1e12
    roof = {"bound": peak["bound"], "achieved": achieved, "peak": peak["peak"],
            "unit": peak["unit"], "frac": achieved / peak["peak"],
            "traffic": load_traffic(args.workload, args.algo), "kernel_ms": kern_avg,
            "pack_ms_est": statistics.mean(pack_ms), "peak_source": peak["peak_source"],
            "ops_per_launch": ops, "popc_pipe_peak_tops": peak["popc_peak"]}
    if "cublas_int8_tops" in peak:
        roof["cublas_int8_tops"] = peak["cublas_int8_tops"]
    if is_net:
        roof["note"] = ("whole-network step: achieved = binary ops of all binary layers / step "
                        "time (float stem / classifier / BN / pooling included in the time)")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.workload)

    if rank == 0:
        line = {
            "metric": metric, "value": value, "unit": unit, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": (("b1 planes -> u8 (tcgen05 kind::i8), s32" if args.workload.endswith("2bit")
                       else DTYPE) if args.algo in ("auto", "umma") else "u32 (xor/popc words)"),
            "data": "synthetic (seeded, BASELINE.json shapes)",
            "config": {"workload": d["workload"], "M": d["M"], "N": d["N"], "K": d["K"],
                       "batch_per_gpu": d["batch"], "parallelism": f"replicas x{world}",
                       "l2": "flushed between timed steps (256 MiB write, then 256 MiB read so the "
                             "write-backs land outside the timed region)",
                       "launch": "CUDA graph per step (pack + kernel)",
                       "algo": args.algo},
            "e2e": e2e, "gpu_launches": plan.launches_per_step * args.steps,
            "roofline": roof, "cpu_baseline": cpu, "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_gpu_arm(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()

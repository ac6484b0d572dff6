#!/usr/bin/env python
"""Benchmark of the B200 binarise -> bit-pack -> xnor-popcount hot path.

Default workload = BASELINE.json configs[3]: binary ResNet-18 inference,
256 x 3 x 224 x 224 f32 ~ N(0,1) images, random-init weights, batch-sharded
across the GPUs (metric: images/s).  A step = the whole ``infer_packed``
forward of the resident batch (float stem, every binary conv with its fused
BN / sign-pack epilogue, residual adds, classifier head), one CUDA graph.
Other workloads: ``c2`` (configs[1], QConvolution 3x3 256->256 on
32x256x28x28, binary TOPS = 2MNK / step), ``c1`` (configs[0] QFullyConnected),
``gemm4096|gemm8192|gemm16384|gemm4096k65536|gemm4096_2bit`` (configs[4]),
``lenet`` (configs[2]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload resnet18|lenet|c2|c1|gemm4096|...]

N > 1: one process per GPU over NCCL (launched by torchrun, or by this script
itself when WORLD_SIZE is unset).  Networks shard the fixed 256 (1024) image
batch over the ranks (``"scaling": "strong"``, BASELINE configs[3]) and also
report the weak-scaling figure (every rank a full batch); configs[4] GEMMs
split N over the ranks and all-gather the output shards (strong); the single
layers c1 / c2 run one replica per rank (weak).  Time = max over ranks.
``--impl reference`` times the reference's CPU algorithm (the pinned oracle
port, oracle/, all host threads) on the same workload; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
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
    p.add_argument("--workload", choices=WORKLOADS, default="resnet18")
    p.add_argument("--algo", default="auto")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    # test hook: gloo ranks sharing the visible GPU(s) (host-staged gathers; no kernel
    # waits on another rank) to exercise the N > 1 code paths on a one-GPU box
    p.add_argument("--backend", choices=("nccl", "gloo"), default="nccl")
    return p.parse_args()


# ----------------------------------------------------------------- workloads
SCALING = {"resnet18": "strong", "lenet": "strong", "gemm4096": "strong", "gemm8192": "strong",
           "gemm16384": "strong", "gemm4096k65536": "strong", "gemm4096_2bit": "strong",
           "c1": "weak", "c2": "weak"}


def workload_desc(name):
    import workloads as wl
    if name in NET_WORKLOADS:
        desc, batch, chw = NET_WORKLOADS[name]
        return dict(workload=desc + f", batch {batch} " + ("U[0,1]" if name == "lenet" else "N(0,1)")
                    + f" images {chw}, random-init weights",
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


def build_plan(name, algo, world=1, rank=0, weak=False):
    """The workload's plan for this rank.  Networks: this rank's batch shard (strong
    scaling; ``weak`` = a full batch per rank); configs[4] GEMMs at world > 1: this
    rank's N shard + all-gather; c1 / c2: one full replica per rank."""
    import torch

    import workloads as wl
    import paper_1705_09864_b200 as bnn
    from paper_1705_09864_b200.parallel import shard_bounds
    from paper_1705_09864_b200.plan import ConvPlan, DensePlan, GemmPlan, NsplitGemmPlan

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
        b0, b1 = (0, batch) if weak else shard_bounds(batch, world, rank)[:2]
        net = nets.lenet_c3(d["seed"]) if name == "lenet" else nets.resnet18_c4(d["seed"])
        net.pack_for_inference()
        g = torch.Generator(device="cuda").manual_seed(d["seed"])
        full = (torch.rand if name == "lenet" else torch.randn)((batch,) + chw, device="cuda",
                                                             generator=g)
        plan = NetPlan(net, b1 - b0, chw)
        plan.x.copy_(full[b0:b1])
        del full
        return plan, plan.x.cpu().pin_memory()
    if name.endswith("_2bit"):
        from paper_1705_09864_b200.bitpack import pack_planes_device
        from paper_1705_09864_b200.plan import BitplanePlan
        g = torch.Generator(device="cuda").manual_seed(d["seed"])
        wf = torch.rand((d["M"], d["K"]), device="cuda", generator=g)
        xf = torch.rand((d["N"], d["K"]), device="cuda", generator=g)
        ap = pack_planes_device(wf, 2, "unsigned")
        bp = pack_planes_device(xf, 2, "unsigned")
        if world > 1:
            from paper_1705_09864_b200.gemm import bitplane_gemm
            n0, n1, _ = shard_bounds(d["N"], world, rank)
            bs = bp[:, n0:n1].contiguous()

            def compute(a_, b_, k_, out):
                bitplane_gemm(a_, b_, k_, a_grid="unsigned", b_grid="unsigned", out=out,
                              transpose_out=True)
            plan = NsplitGemmPlan(ap, bs, d["K"], d["N"], algo=algo)
            plan.ns._compute = compute
            return plan, bs.cpu().pin_memory()
        return BitplanePlan(ap, bp, d["K"]), bp.cpu().pin_memory()
    g = torch.Generator(device="cuda").manual_seed(d["seed"])
    W = (d["K"] + 63) // 64
    aw = torch.randint(-2**63, 2**63 - 1, (d["M"], W), device="cuda", generator=g).view(torch.uint64)
    bw = torch.randint(-2**63, 2**63 - 1, (d["N"], W), device="cuda", generator=g).view(torch.uint64)
    if world > 1:
        n0, n1, _ = shard_bounds(d["N"], world, rank)
        bs = bw[n0:n1].clone()
        del bw
        return NsplitGemmPlan(aw, bs, d["K"], d["N"], algo=algo), bs.cpu().pin_memory()
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
        "higher_is_better": True,
        "scaling": SCALING[name] if args.gpus > 1 else ("strong" if is_net else "weak"),
        "vs_baseline": None, "dtype": "u64 (xor / popcount words)",
        "data": "synthetic (seeded, BASELINE.json shapes)",
        # the same config keys and workload as the GPU arm
        "config": {"workload": d["workload"], "M": d["M"], "N": d["N"], "K": d["K"],
                   "batch_per_gpu": d["batch"],
                   "parallelism": f"{os.cpu_count()} host threads (rank 0 only)",
                   "l2": "n/a (host)", "launch": "host calls", "algo": "reference CPU port"},
        "cpu_baseline": {"value": value, "unit": unit, "cores": os.cpu_count(), "kind": "port",
                         "sample": desc + " (the oracle/ C port of the reference composition; "
                                          "the Python/numba reference itself cannot travel to "
                                          "the GPU box and is ~8x slower, so this arm is "
                                          "conservative)"},
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
        # every workload's dominant kernel runs kind::mxf4: on bits expanded in SMEM (convs, small
        # GEMMs), or -- configs[4], 1-bit and 2-bit -- on operands pre-expanded to e2m1 values in
        # HBM by a pass that is part of the timed step (bnn_gemm_xp.cu, 2-CTA pairs)
        kind = "mxf4"
        how = ("operands expanded once per step to e2m1 values in HBM, 2-CTA TMA-fed GEMM "
               "(bnn_gemm_xp.cu; the expansion pass is inside kernel_ms)"
               if workload.startswith("gemm") else "bits expanded in SMEM")
        return {"bound": "tensor", "peak": tcgen05_peak_tops(kind), "unit": "TOPS",
                "peak_source": f"measured: dense tcgen05.mma kind::{kind} issue rate, one CTA per "
                               "SM, 128x256 MMAs back to back (bnn_probe_pipe_peak); the engine "
                               f"runs kind::{kind} on {how}",
                "popc_peak": popc, "cublas_int8_tops": int8_tensor_peak_tops()}
    return {"bound": "popc", "peak": popc, "unit": "TOPS",
            "peak_source": "measured: bnn_probe_pipe_peak POPC rate x 64 binary ops "
                           "(32 bits x {xor, add})", "popc_peak": popc}


def _graphs(plan):
    """(step graph, kernel-only graph) or (None, None) for plans whose step holds a
    collective (replayed eagerly)."""
    import torch
    if not getattr(plan, "graph_ok", True):
        return None, None
    stream = torch.cuda.current_stream()
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
    return g_step, g_kern


def _timed_steps(step, steps, l2_flush, world, sampler=None):
    """Per-step CUDA-event times (ms) on the launching stream, L2 flushed between steps
    outside the events; barrier + synchronize on both sides of the timed region."""
    import torch
    import torch.distributed as dist
    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if sampler is not None:
        sampler.__enter__()
    try:
        for i in range(steps):
            l2_flush()
            s, e = ev[i]
            s.record(stream)
            step()
            e.record(stream)
        torch.cuda.synchronize()
    finally:
        if sampler is not None:
            sampler.__exit__(None, None, None)
    if world > 1:
        dist.barrier()
    return [s.elapsed_time(e) for s, e in ev]


def _max_over_ranks(v, world):
    import torch
    import torch.distributed as dist
    if world == 1:
        return v
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _kernel_families(plan):
    """Per-family device time of one network step (NetPlan.kernel_breakdown): the binary
    convs / GEMMs (xnor_umma_kernel), the float stem, the rest of this library's kernels."""
    fam = {}
    for name, ms, ops in plan.kernel_breakdown():
        if name.startswith(("bnn_bconv2d", "bnn_xnor_gemm")):
            key = "binary conv / GEMM (xnor_wconv / xnor_sconv / xconv_xp / xnor_umma / xnor_pw kernels)"
        elif "f32_tc" in name:
            key = "float stem (stem_s2_kernel / conv_pool_kernel, tcgen05 kind::tf32 split)"
        else:
            key = "other (" + name + ")"
        f = fam.setdefault(key, {"ms": 0.0, "launches": 0, "binary_ops": 0})
        f["ms"] += ms
        f["launches"] += 1
        f["binary_ops"] += ops
    return fam


def _stem_roofline(fams, batch):
    """The float stem's own roofline (the second-largest share of the ResNet-18 step): tensor
    cores, kind::tf32.  bnn_stem_s2.cu issues 2 x 21 MMAs of 128 x 112 x 8 per conv row (four
    hi/lo split products on a K padded from 147 to 168) for 4 bands x 29 rows per image; peak =
    half the measured dense bf16 rate of MEASURED_PEAKS.json (TF32 runs at half the bf16 rate;
    tools/probes/tf32_overlap.cu measures 2,048 MAC/clk/SM), else the B200 nominal 1.1 PFLOP/s."""
    ms = sum(v["ms"] for k, v in fams.items() if k.startswith("float stem"))
    issued = 2.0 * 2 * 21 * 128 * 112 * 8 * (4 * 29) * batch
    algorithmic = 2.0 * 64 * 147 * 112 * 112 * batch
    peak, src = 1100.0, "fallback: B200 nominal dense TF32"
    try:
        pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        peak, src = pk["bf16_tflops"] / 2, "MEASURED_PEAKS.json bf16_tflops (burst) / 2"
    except Exception:
        pass
    ach = issued / (ms * 1e-3) / 1e12
    return {"bound": "tensor", "kernel": "stem_s2_kernel (tcgen05 kind::tf32)", "kernel_ms": ms,
            "achieved": ach, "peak": peak, "unit": "TFLOP/s (TF32 MMA flops issued)", "frac": ach / peak,
            "algorithmic_f32_tflops": algorithmic / (ms * 1e-3) / 1e12, "peak_source": src}


def run_gpu_arm(args, rank, world, local_rank):
    import torch

    torch.cuda.set_device(local_rank % torch.cuda.device_count())
    import paper_1705_09864_b200 as bnn
    bnn.load_library()

    name = args.workload
    is_net = name in NET_WORKLOADS
    scaling = SCALING[name] if world > 1 else ("strong" if is_net else "weak")
    plan, host_x = build_plan(name, args.algo, world, rank)
    d = workload_desc(name)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MiB > L2
    flush_rd = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    flush_sink = torch.empty((), dtype=torch.float32, device="cuda")

    def l2_flush():
        # write a buffer larger than L2 (evicts every line of this step's data), then
        # read another one so the dirty lines of the write are written back here, outside
        # the timed region, instead of inside the next timed kernel
        flush.zero_()
        torch.amax(flush_rd, dim=0, out=flush_sink)

    # each step is one CUDA-graph replay (the GPU work only); the kernel alone is a second
    # graph, timed the same way, for the roofline.  Plans whose step holds a collective
    # (N-split GEMM at world > 1) run eagerly.
    g_step, g_kern = _graphs(plan)
    step = g_step.replay if g_step is not None else plan.run_device
    kern = g_kern.replay if g_kern is not None else plan.kernel
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clk = ClockSampler(local_rank % torch.cuda.device_count())
    step_ms = _timed_steps(step, args.steps, l2_flush, world, clk)
    kern_ms = _timed_steps(kern, args.steps, l2_flush, world)
    plan.check_flags()
    total_ms = _max_over_ranks(sum(step_ms), world)
    ms_per_step = total_ms / args.steps
    units = d["batch"] if is_net else plan.binary_ops / 1e12  # whole-job images or tera-ops
    if scaling == "weak" and world > 1:
        units *= world  # every rank ran a full replica
    metric = NET_WORKLOADS[name][0] if is_net else METRIC
    unit = "images/s" if is_net else UNIT
    value = units / (ms_per_step * 1e-3)

    gather = None
    if isinstance(plan, _nsplit_type()):
        # the collective alone (the step is GEMM + all-gather)
        gms = _timed_steps(plan.ns.gather, args.steps, lambda: None, world)
        gather = {"ms_per_step": _max_over_ranks(statistics.mean(gms), world),
                  "bytes_per_rank": plan.ns.full.numel() * 4,
                  "what": "torch.distributed.all_gather_into_tensor (NCCL) of the [N/g, M] f32 "
                          "output shards"}

    # end to end through the public plan API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        y_host = torch.empty(plan.y.shape, dtype=plan.y.dtype).pin_memory()
        for _ in range(2):
            plan.run_host(host_x, y_host)
        import torch.distributed as dist
        if world > 1:
            dist.barrier()
        stream = torch.cuda.current_stream()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0.record(stream)
        for _ in range(args.steps):
            plan.run_host(host_x, y_host)
        t1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = _max_over_ranks(t0.elapsed_time(t1), world) / args.steps
        e2e = {"value": units / (e2e_ms * 1e-3), "unit": unit,
               "h2d_bytes_per_step": plan.h2d_bytes, "d2h_bytes_per_step": plan.d2h_bytes,
               "ms_per_step": e2e_ms,
               "path": (f"{type(plan).__name__}.run_host: pinned H2D -> pack -> kernels -> "
                        "D2H -> sync (one CUDA-graph replay per call, pipelined over "
                        f"{getattr(plan, 'host_chunks', 1)} batch slices on 3 streams; the slice count is "
                        "tuned once on the first call, outside the timed region)")
               if getattr(plan, "graph_ok", True) else
               (f"{type(plan).__name__}.run_host: pinned H2D of this rank's packed B shard -> "
                "GEMM -> all-gather -> D2H of the full result -> sync (eager)")}

    # weak-scaling companion of a strong-scaled network (every rank a full batch)
    weak = None
    if is_net and world > 1:
        wplan, _ = build_plan(name, args.algo, world, rank, weak=True)
        wg, _ = _graphs(wplan)
        for _ in range(args.warmup):
            wg.replay()
        wms = _timed_steps(wg.replay, args.steps, l2_flush, world)
        w_ms = _max_over_ranks(sum(wms), world) / args.steps
        weak = {"value": world * d["batch"] / (w_ms * 1e-3), "unit": unit, "ms_per_step": w_ms,
                "batch_per_gpu": d["batch"]}
        del wplan, wg

    kern_avg = statistics.mean(kern_ms)
    ops_rank = getattr(plan, "local_ops", plan.binary_ops)
    if is_net:
        fams = _kernel_families(plan)
        step_dev = sum(f["ms"] for f in fams.values())
        key = "binary conv / GEMM (xnor_wconv / xnor_sconv / xconv_xp / xnor_umma / xnor_pw kernels)"
        bf = fams[key]
        peak = pipe_peak(args.algo, name)
        achieved = bf["binary_ops"] / (bf["ms"] * 1e-3) / 1e12
        roof = {"bound": peak["bound"], "achieved": achieved, "peak": peak["peak"],
                "unit": peak["unit"], "frac": achieved / peak["peak"],
                "traffic": load_traffic(name, args.algo),
                "kernel": key + f": {bf['launches']} launches per step",
                "kernel_ms": bf["ms"], "ops_per_step": bf["binary_ops"],
                "share_of_step": bf["ms"] / step_dev,
                "families": {k: dict(v, share=v["ms"] / step_dev) for k, v in fams.items()},
                "peak_source": peak["peak_source"], "popc_pipe_peak_tops": peak["popc_peak"],
                "note": "per-launch CUDA events of one eager step queued behind a sleep kernel "
                        "(no host gaps inside the intervals); achieved = 2MNK of every binary "
                        "conv / GEMM launch / their summed device time"}
        if roof["traffic"]:
            # the same family against HBM: the layer-1/2 convs that stream an f32 shortcut in and
            # an f32 block output out are bound by that stream, not by the tensor pipe
            try:
                hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
                src = "MEASURED_PEAKS.json hbm_gbs"
            except Exception:
                hbm, src = 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s measured on this pool)"
            gbs = roof["traffic"] / (bf["ms"] * 1e-3) / 1e9
            roof["hbm"] = {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s",
                           "frac": gbs / hbm, "peak_source": src,
                           "note": "ncu DRAM bytes of the family per step (profiles/traffic.json) / "
                                   "its summed device time"}
        if name == "resnet18":
            roof["stem"] = _stem_roofline(fams, plan.b)
    else:
        peak = pipe_peak(args.algo, name)
        achieved = ops_rank / (kern_avg * 1e-3) / 1e12
        roof = {"bound": peak["bound"], "achieved": achieved, "peak": peak["peak"],
                "unit": peak["unit"], "frac": achieved / peak["peak"],
                "traffic": load_traffic(name, args.algo), "kernel_ms": kern_avg,
                "pack_ms_est": statistics.mean(max(0.0, a - b) for a, b in zip(step_ms, kern_ms)),
                "peak_source": peak["peak_source"], "ops_per_launch": ops_rank,
                "popc_pipe_peak_tops": peak["popc_peak"]}
    if "cublas_int8_tops" in peak:
        roof["cublas_int8_tops"] = peak["cublas_int8_tops"]

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(name)

    if rank == 0:
        if is_net:
            par = f"batch-sharded dp{world} ({plan.b} images per GPU)" if world > 1 \
                else f"1 GPU, batch {plan.b}"
        elif scaling == "strong" and world > 1:
            par = f"N split over {world} GPUs + NCCL all-gather of the output shards"
        else:
            par = f"replicas x{world}"
        line = {
            "metric": metric, "value": value, "unit": unit, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
            "dtype": (("2-bit codes -> e2m1 grid values (tcgen05 kind::mxf4), exact f32 numerator"
                       if name.endswith("2bit")
                       else DTYPE) if args.algo in ("auto", "umma") else "u32 (xor/popc words)"),
            "data": "synthetic (seeded, BASELINE.json shapes)",
            "config": {"workload": d["workload"], "M": d["M"], "N": d["N"], "K": d["K"],
                       "batch_per_gpu": plan.b if is_net else d["batch"], "parallelism": par,
                       "l2": "flushed between timed steps (256 MiB write, then 256 MiB read so the "
                             "write-backs land outside the timed region)",
                       "launch": "CUDA graph per step" if g_step is not None else
                                 "eager step (kernel + collective)",
                       "algo": args.algo},
            "e2e": e2e, "gpu_launches": plan.launches_per_step * args.steps,
            "roofline": roof, "cpu_baseline": cpu, "clocks": clk.summary(),
        }
        if weak is not None:
            line["weak_scaling"] = weak
        if gather is not None:
            line["gather"] = gather
        print(json.dumps(line), flush=True)


def _nsplit_type():
    from paper_1705_09864_b200.plan import NsplitGemmPlan
    return NsplitGemmPlan


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn_ranks(args) -> int:
    """``bench.py --gpus N`` without a torchrun environment: launch N ranks (one process
    per GPU) through torch.distributed.run on 127.0.0.1 and return its exit code; rank 0
    prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl != "reference":
        sys.exit(spawn_ranks(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if args.backend == "nccl":
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group("gloo")
    try:
        run_gpu_arm(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""xnor-popcount GEMM on the B200 and its benchmark harness.

Drop-in for the reference ``bitnn.gemm`` (``/root/reference/pkg/src/bitnn/
gemm.py``): the public kernels take two ``BitMatrix`` operands (layouts 'a'
and 'b', complementary tails), validate them exactly like ``_check_operands``
(gemm.py:212-223) and return the popcount-domain product as float32 [M, N].
All reference kernel ids (``xnor_base`` ... ``xnor_parallel``) run the same
CUDA engine here -- on a GPU there is one kernel, selected by ``algo`` --
plus the new id ``xnor_b200``.  ``workers`` / ``BMX_THREADS`` keep their
meaning for the CPU-thread count contract only (validated, then ignored).
"""

from __future__ import annotations

import os
import statistics
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .bitpack import BitMatrix, binarize, pack_matrix_a, pack_matrix_b, words_per_bits

THREADS_ENV_VAR = "BMX_THREADS"
MAX_K_EXACT = 1 << 24  # gemm.py:43-44
DEFAULT_BLOCK_ROWS = 32
DEFAULT_BLOCK_WORDS = 512
CSV_HEADER = "kernel,M,N,K,repeats,median_ns,pack_ns,checksum,seed"  # gemm.py:49


@dataclass(frozen=True)
class GemmDims:
    """gemm.GemmDims (gemm.py:162-189)."""

    m: int
    n: int
    k: int

    def __post_init__(self):
        if min(self.m, self.n, self.k) < 1:
            raise ValueError(f"GEMM dims must be positive, got {self}")
        if self.k >= MAX_K_EXACT:
            raise ValueError(f"K={self.k} exceeds {MAX_K_EXACT - 1}; popcounts would lose "
                             "exactness in float32 outputs")

    @property
    def words_per_k(self) -> int:
        return words_per_bits(self.k)

    @property
    def operand_bytes(self) -> int:
        floats = 4 * (self.m * self.k + self.k * self.n)
        packed = 8 * self.words_per_k * (self.m + self.n)
        return floats + packed + 4 * self.m * self.n

    @property
    def binary_ops(self) -> int:
        """2*M*N*K, the metric's unit of work (BASELINE.json)."""
        return 2 * self.m * self.n * self.k


def resolve_workers(explicit=None) -> int:
    """gemm.resolve_workers (gemm.py:192-209): explicit > BMX_THREADS > cpu_count."""
    if explicit is not None:
        workers = int(explicit)
    else:
        env = os.environ.get(THREADS_ENV_VAR)
        if env is not None:
            try:
                workers = int(env)
            except ValueError:
                raise ValueError(f"{THREADS_ENV_VAR} must be a positive integer, got {env!r}") from None
        else:
            workers = os.cpu_count() or 1
    if workers < 1:
        raise ValueError(f"worker count must be positive, got {workers}")
    return workers


def _check_operands(a: BitMatrix, b: BitMatrix) -> None:
    """gemm._check_operands (gemm.py:212-223) minus the host allocation."""
    if a.layout != "a" or b.layout != "b":
        raise ValueError(f"operand layouts must be ('a', 'b'), got ({a.layout!r}, {b.layout!r})")
    if a.pad_fill != 0 or b.pad_fill != 1:
        raise ValueError("operands must use complementary padding (a: 0, b: 1)")
    if a.n_bits != b.n_bits:
        raise ValueError(f"reduction lengths differ: {a.n_bits} vs {b.n_bits}")
    GemmDims(a.vectors, b.vectors, a.n_bits)


# ----------------------------------------------------------------- device GEMM
def xnor_rows_gemm(a_rows: torch.Tensor, b_rows: torch.Tensor, k: int, *, a_pad: int = 0,
                   b_pad: int = 0, domain: int = _lib.POPCOUNT, out: torch.Tensor | None = None,
                   transpose_out: bool = False, scale: torch.Tensor | None = None,
                   shift: torch.Tensor | None = None, algo: int | str = "auto",
                   workspace_in: torch.Tensor | None = None) -> torch.Tensor:
    """Core entry: both operands K-contiguous [M, W] / [N, W] CUDA u64 words.

    Returns f32 [M, N] (or [N, M] with ``transpose_out``), popcount domain
    unless ``domain == DOT``.  Asynchronous on the current stream.
    """
    if isinstance(algo, str):
        algo = _lib.ALGOS[algo]
    m, n = a_rows.shape[0], b_rows.shape[0]
    GemmDims(m, n, k)
    if a_rows.stride(1) != 1 or b_rows.stride(1) != 1:
        raise ValueError("word rows must be contiguous")
    if out is None:
        out = torch.empty((n, m) if transpose_out else (m, n), dtype=torch.float32,
                          device=a_rows.device)
    ldc_m, ldc_n = (1, out.stride(0)) if transpose_out else (out.stride(0), 1)
    if scale is None and shift is None and (algo == _lib.ALGO_UMMA_XP or
                                            (algo == _lib.ALGO_AUTO and xp_eligible(m, n, k))):
        # large GEMMs: operands expanded once into a scratch buffer, 2-CTA TMA-fed engine
        ws = workspace(m, n, k, a_rows.device) if workspace_in is None else workspace_in
        _lib.call("bnn_xnor_gemm_ws", _lib.ptr(a_rows), a_rows.stride(0), _lib.ptr(b_rows),
                  b_rows.stride(0), m, n, k, a_pad, b_pad, _lib.ptr(out), ldc_m, ldc_n, domain,
                  algo, _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
        return out
    _lib.call("bnn_xnor_gemm", _lib.ptr(a_rows), a_rows.stride(0), _lib.ptr(b_rows),
              b_rows.stride(0), m, n, k, a_pad, b_pad, _lib.ptr(out), ldc_m, ldc_n, domain,
              _lib.ptr(scale), _lib.ptr(shift), algo, _lib.stream_ptr())
    return out


def xp_eligible(m: int, n: int, k: int) -> bool:
    """Shapes AUTO hands to the pre-expanded engine when a workspace comes with the call
    (mirrors xp_auto in csrc/bnn_capi.cu)."""
    return m >= 1024 and n >= 1024 and k >= 2048 and float(m) * n * k >= 3.0e10


_WORKSPACES: dict = {}


def scratch(need: int, device) -> torch.Tensor:
    """One growing u8 buffer per (device, stream) for the pre-expanded engines -- calls on one
    stream are ordered, so they can share it."""
    key = (torch.device(device).index, int(torch.cuda.current_stream().cuda_stream))
    ws = _WORKSPACES.get(key)
    if ws is None or ws.numel() < need:
        ws = torch.empty(need, dtype=torch.uint8, device=device)
        _WORKSPACES[key] = ws
    return ws


def workspace(m: int, n: int, k: int, device) -> torch.Tensor:
    """Scratch for bnn_xnor_gemm_ws / bnn_bitplane_gemm_ws."""
    return scratch(int(_lib.load().bnn_xnor_gemm_ws_bytes(m, n, k)), device)


def bitplane_gemm(a_planes: torch.Tensor, b_planes: torch.Tensor, k: int, *,
                  a_grid: str = "signed", b_grid: str = "signed", out: torch.Tensor | None = None,
                  transpose_out: bool = False, algo: int | str = "auto",
                  workspace_in: torch.Tensor | None = None) -> torch.Tensor:
    """Multi-bit (bit-plane) GEMM: sum_k v_a v_b for [bits, M, W] x [bits, N, W] planes.

    The product the reference's float path computes for bits > 1
    (layers.py:240-242, 370-377); exact integer numerator, one f32 rounding.
    """
    bits, m, w = a_planes.shape
    bits_b, n, w2 = b_planes.shape
    if bits != bits_b or w != w2:
        raise ValueError("plane counts or word counts differ")
    GemmDims(m, n, k)
    if out is None:
        out = torch.empty((n, m) if transpose_out else (m, n), dtype=torch.float32,
                          device=a_planes.device)
    ldc_m, ldc_n = (1, out.stride(0)) if transpose_out else (out.stride(0), 1)
    g = {"signed": _lib.GRID_SIGNED, "unsigned": _lib.GRID_UNSIGNED}
    if isinstance(algo, str):
        algo = _lib.ALGOS[algo]
    if algo == _lib.ALGO_UMMA_XP or (algo == _lib.ALGO_AUTO and xp_eligible(m, n, k)):
        # large shapes: code values as e2m1 numbers in a scratch buffer, 2-CTA TMA-fed engine
        ws = workspace(m, n, k, a_planes.device) if workspace_in is None else workspace_in
        _lib.call("bnn_bitplane_gemm_ws", _lib.ptr(a_planes), w, m * w, g[a_grid], _lib.ptr(b_planes),
                  w, n * w, g[b_grid], bits, m, n, k, _lib.ptr(out), ldc_m, ldc_n, algo, _lib.ptr(ws),
                  ws.numel(), _lib.stream_ptr())
        return out
    _lib.call("bnn_bitplane_gemm", _lib.ptr(a_planes), w, m * w, g[a_grid], _lib.ptr(b_planes), w,
              n * w, g[b_grid], bits, m, n, k, _lib.ptr(out), ldc_m, ldc_n, _lib.stream_ptr())
    return out


def xnor_gemm_b200(a: BitMatrix, b: BitMatrix, algo: int | str = "auto",
                   domain: int = _lib.POPCOUNT) -> torch.Tensor:
    """Packed product of a layout-'a' and a layout-'b' operand: f32 [M, N] on the GPU."""
    _check_operands(a, b)
    return xnor_rows_gemm(a.words, b.rows(), a.n_bits, a_pad=a.pad_fill, b_pad=b.pad_fill,
                          domain=domain, algo=algo)


def _host(c: torch.Tensor) -> np.ndarray:
    return c.cpu().numpy()


def xnor_gemm_base(a: BitMatrix, b: BitMatrix) -> np.ndarray:
    """gemm.xnor_gemm_base (gemm.py:226-230) contract; B200 engine."""
    return _host(xnor_gemm_b200(a, b))


def xnor_gemm_blocked(a: BitMatrix, b: BitMatrix, block_rows: int = DEFAULT_BLOCK_ROWS,
                      block_words: int = DEFAULT_BLOCK_WORDS) -> np.ndarray:
    """gemm.xnor_gemm_blocked (gemm.py:233-244): tile args validated; output unchanged."""
    if block_rows < 1 or block_words < 1:
        raise ValueError("tile sizes must be positive")
    return _host(xnor_gemm_b200(a, b))


def xnor_gemm_unrolled(a: BitMatrix, b: BitMatrix) -> np.ndarray:
    """gemm.xnor_gemm_unrolled (gemm.py:247-251)."""
    return _host(xnor_gemm_b200(a, b))


def xnor_gemm_parallel(a: BitMatrix, b: BitMatrix, workers=None,
                       block_rows: int = DEFAULT_BLOCK_ROWS,
                       block_words: int = DEFAULT_BLOCK_WORDS) -> np.ndarray:
    """gemm.xnor_gemm_parallel (gemm.py:254-284): the GPU grid replaces the thread pool."""
    if block_rows < 1 or block_words < 1:
        raise ValueError("tile sizes must be positive")
    resolve_workers(workers)
    return _host(xnor_gemm_b200(a, b))


def xnor_gemm_base_soft(a: BitMatrix, b: BitMatrix) -> np.ndarray:
    """gemm.xnor_gemm_base_soft (gemm.py:287-291)."""
    return _host(xnor_gemm_b200(a, b))


KERNEL_IDS = ("naive_f32", "xnor_base", "xnor_blocked", "xnor_unrolled", "xnor_parallel",
              "xnor_b200")


def gemm_f32(a, b) -> np.ndarray:
    """tensor.gemm_f32 (tensor.py:116-131) float baseline, on the GPU (TF32 off)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    if a.ndim != 2 or b.ndim != 2:
        raise ValueError("gemm_f32 expects 2-D operands")
    if a.shape[1] != b.shape[0]:
        raise ValueError(f"inner dimensions differ: {a.shape} @ {b.shape}")
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        c = torch.from_numpy(a).cuda() @ torch.from_numpy(b).cuda()
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return c.cpu().numpy()


def run_kernel(kernel: str, a_f32, b_f32, a_bm=None, b_bm=None, **kw) -> np.ndarray:
    """gemm.run_kernel (gemm.py:297-324): xnor ids return the popcount domain."""
    if kernel == "naive_f32":
        return gemm_f32(a_f32, b_f32)
    if kernel not in KERNEL_IDS:
        raise ValueError(f"unknown kernel {kernel!r}; choose from {KERNEL_IDS}")
    if a_bm is None:
        a_bm = pack_matrix_a(a_f32)
    if b_bm is None:
        b_bm = pack_matrix_b(b_f32)
    if kernel == "xnor_blocked":
        return xnor_gemm_blocked(a_bm, b_bm, kw.get("block_rows", DEFAULT_BLOCK_ROWS),
                                 kw.get("block_words", DEFAULT_BLOCK_WORDS))
    if kernel == "xnor_parallel":
        return xnor_gemm_parallel(a_bm, b_bm, kw.get("workers"))
    return _host(xnor_gemm_b200(a_bm, b_bm, algo=kw.get("algo", "auto")))


# ----------------------------------------------------------------- bench harness
@dataclass
class BenchRecord:
    """gemm.BenchRecord (gemm.py:327-345); field order = CSV schema."""

    kernel: str
    m: int
    n: int
    k: int
    repeats: int
    median_ns: int
    pack_ns: int
    checksum: int
    seed: int

    def to_csv_row(self) -> str:
        return (f"{self.kernel},{self.m},{self.n},{self.k},{self.repeats},"
                f"{self.median_ns},{self.pack_ns},{self.checksum},{self.seed}")


def records_to_csv(records) -> str:
    lines = [CSV_HEADER]
    lines.extend(r.to_csv_row() for r in records)
    return "\n".join(lines) + "\n"


def make_operands(dims: GemmDims, seed: int):
    """gemm.make_operands (gemm.py:354-360): seeded +-1 float32 operands."""
    rng = np.random.default_rng(seed)
    choices = np.array([-1.0, 1.0], dtype=np.float32)
    return rng.choice(choices, size=(dims.m, dims.k)), rng.choice(choices, size=(dims.k, dims.n))


def checksum_popcount(c, kernel: str, dims: GemmDims) -> int:
    """gemm.checksum_popcount (gemm.py:363-373)."""
    c = c.cpu().numpy() if isinstance(c, torch.Tensor) else np.asarray(c)
    total = float(c.sum(dtype=np.float64))
    if kernel == "naive_f32":
        total = (total + float(dims.m) * dims.n * dims.k) / 2.0
    return int(round(total))


def _cuda_time_ns(fn, warmup: int, repeats: int):
    for _ in range(warmup):
        fn()
    samples = []
    out = None
    for _ in range(repeats):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        out = fn()
        e.record()
        e.synchronize()
        samples.append(int(s.elapsed_time(e) * 1e6))
    return samples, out


def benchmark_kernel(kernel: str, dims: GemmDims, repeats: int = 5, warmup: int = 1,
                     seed: int = 0, block_rows: int = DEFAULT_BLOCK_ROWS,
                     block_words: int = DEFAULT_BLOCK_WORDS, workers=None,
                     algo: str = "auto") -> BenchRecord:
    """gemm.benchmark_kernel (gemm.py:376-428), timed with CUDA events.

    ``pack_ns`` covers binarize + pack of the right operand (activation side);
    the left operand is packed outside the clock, as deployed weights are.
    """
    if kernel not in KERNEL_IDS:
        raise ValueError(f"unknown kernel {kernel!r}; choose from {KERNEL_IDS}")
    if repeats < 1 or warmup < 0:
        raise ValueError("repeats must be >= 1 and warmup >= 0")
    a_f32, b_f32 = make_operands(dims, seed)
    if kernel == "naive_f32":
        at, bt = torch.from_numpy(a_f32).cuda(), torch.from_numpy(b_f32).cuda()
        prev = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = False
        try:
            samples, c = _cuda_time_ns(lambda: at @ bt, warmup, repeats)
        finally:
            torch.backends.cuda.matmul.allow_tf32 = prev
        pack_ns = 0
    else:
        from .bitpack import pack_rows_device

        a_bm = pack_matrix_a(a_f32)
        bt = torch.from_numpy(np.ascontiguousarray(b_f32.T)).cuda()  # activations [N, K]
        psamples, b_rows = _cuda_time_ns(lambda: pack_rows_device(bt, 0), 1, 1)
        pack_ns = psamples[0]
        samples, c = _cuda_time_ns(
            lambda: xnor_rows_gemm(a_bm.words, b_rows, dims.k, a_pad=0, b_pad=0, algo=algo),
            warmup, repeats)
    torch.cuda.synchronize()
    return BenchRecord(kernel=kernel, m=dims.m, n=dims.n, k=dims.k, repeats=repeats,
                       median_ns=int(statistics.median(samples)), pack_ns=pack_ns,
                       checksum=checksum_popcount(c, kernel, dims), seed=seed)

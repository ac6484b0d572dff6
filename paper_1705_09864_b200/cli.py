"""``python -m paper_1705_09864_b200 bench gemm|conv`` -- the reference's bench CLI
(``bitnn bench``, cli.py:139-156 parser, :252-320 run) on the B200 kernels.

Same arguments, same frozen CSV on stdout (``kernel,M,N,K,repeats,median_ns,pack_ns,
checksum,seed``, gemm.py:49), same guard: when the kernels' checksums disagree the
command exits 3 (EXIT_INTERNAL, cli.py:276-280).  Every kernel id runs the GPU
engine its name maps to (``gemm.run_kernel``); ``naive_f32`` is the float GEMM of
the +-1 operands (the reference's BLAS baseline), timed on the GPU too.  Per row,
stderr gets a ``#`` comment with binary TOPS (2MNK / median) and the fraction of
the measured tcgen05 kind::mxf4 MMA issue rate (the roofline of DESIGN.md); with
``--extended`` those two numbers are also appended to the CSV rows as
``tops,roofline_frac`` (the default output keeps the frozen schema).
"""

from __future__ import annotations

import argparse
import os
import sys

EXIT_OK, EXIT_USAGE, EXIT_DATA, EXIT_INTERNAL = 0, 1, 2, 3  # cli.py:33-36
MAX_BENCH_BYTES = 8 << 30  # cli.py:39


class UsageError(Exception):
    pass


class InternalCheckError(Exception):
    pass


def build_parser() -> argparse.ArgumentParser:
    from .gemm import DEFAULT_BLOCK_ROWS, DEFAULT_BLOCK_WORDS
    p = argparse.ArgumentParser(prog="python -m paper_1705_09864_b200")
    sub = p.add_subparsers(dest="command", required=True)
    p_bench = sub.add_parser("bench", help="time the GEMM kernels")
    bench_sub = p_bench.add_subparsers(dest="bench_command", required=True)

    def add_common_bench(q):
        q.add_argument("--kernels", default="all", help="comma list of kernel ids, or 'all'")
        q.add_argument("--repeats", type=int, default=5)
        q.add_argument("--warmup", type=int, default=1)
        q.add_argument("--seed", type=int, default=0)
        q.add_argument("--csv", default=None, help="also write records to this file")
        q.add_argument("--block-rows", type=int, default=DEFAULT_BLOCK_ROWS)
        q.add_argument("--block-words", type=int, default=DEFAULT_BLOCK_WORDS)
        q.add_argument("--workers", type=int, default=None)
        q.add_argument("--extended", action="store_true",
                       help="append tops,roofline_frac columns to the CSV rows")

    p_gemm = bench_sub.add_parser("gemm", help="one problem size")
    p_gemm.add_argument("-M", type=int, required=True)
    p_gemm.add_argument("-N", type=int, required=True)
    p_gemm.add_argument("-K", type=int, required=True)
    add_common_bench(p_gemm)
    p_gemm.set_defaults(func=cmd_bench_gemm)

    p_conv = bench_sub.add_parser("conv", help="sweep convolution-shaped problems over input "
                                               "channels")
    p_conv.add_argument("--channels", default="32,64,128,256",
                        help="comma list of input channel counts")
    p_conv.add_argument("--filters", type=int, default=64)
    p_conv.add_argument("--kernel-size", type=int, default=5)
    p_conv.add_argument("--batch", type=int, default=200)
    p_conv.add_argument("--out-hw", type=int, default=8, help="output feature map height and width")
    add_common_bench(p_conv)
    p_conv.set_defaults(func=cmd_bench_conv)
    return p


def _parse_kernels(raw: str):
    from .gemm import KERNEL_IDS
    if raw == "all":
        return list(KERNEL_IDS)
    kernels = [k.strip() for k in raw.split(",") if k.strip()]
    for k in kernels:
        if k not in KERNEL_IDS:
            raise UsageError(f"unknown kernel {k!r}; choose from {', '.join(KERNEL_IDS)}")
    if not kernels:
        raise UsageError("no kernels selected")
    return kernels


_PEAK = []


def mxf4_peak_tops() -> float:
    """Measured dense tcgen05.mma kind::mxf4 issue rate as binary TOPS (2 x MAC/s),
    once per process (bnn_probe_pipe_peak pipe 2)."""
    if not _PEAK:
        import ctypes

        import torch

        from . import _lib
        sink = torch.zeros(1, dtype=torch.int32, device="cuda")
        rate = ctypes.c_double(0)
        _lib.check(_lib.load().bnn_probe_pipe_peak(2, 4096, sink.data_ptr(), ctypes.byref(rate),
                                                   _lib.stream_ptr()), "probe")
        _PEAK.append(2 * rate.value / 1e12)
    return _PEAK[0]


def _run_bench(dims_list, args, out=sys.stdout, err=sys.stderr) -> int:
    from . import gemm
    kernels = _parse_kernels(args.kernels)
    try:
        workers = gemm.resolve_workers(args.workers)
    except ValueError as exc:
        raise UsageError(str(exc)) from None
    if args.repeats < 1 or args.warmup < 0:
        raise UsageError("repeats must be >= 1 and warmup >= 0")
    if args.block_rows < 1 or args.block_words < 1:
        raise UsageError("tile sizes must be positive")
    for dims in dims_list:
        if dims.operand_bytes > MAX_BENCH_BYTES:
            raise UsageError(f"M={dims.m} N={dims.n} K={dims.k} needs about "
                             f"{dims.operand_bytes >> 20} MiB; refusing (limit "
                             f"{MAX_BENCH_BYTES >> 20} MiB)")
    records, extra = [], []
    peak = None
    for dims in dims_list:
        group = [gemm.benchmark_kernel(kernel, dims, repeats=args.repeats, warmup=args.warmup,
                                       seed=args.seed, block_rows=args.block_rows,
                                       block_words=args.block_words, workers=workers)
                 for kernel in kernels]
        if len({r.checksum for r in group}) != 1:
            raise InternalCheckError(f"kernel outputs disagree at M={dims.m} N={dims.n} "
                                     f"K={dims.k}: " + ", ".join(f"{r.kernel}={r.checksum}"
                                                                for r in group))
        records.extend(group)
        for r in group:
            tops = dims.binary_ops / max(r.median_ns, 1) / 1e3
            if peak is None:
                peak = mxf4_peak_tops() if getattr(args, "measure_peak", True) else float("nan")
            extra.append((tops, tops / peak))
            print(f"# M={dims.m} N={dims.n} K={dims.k} {r.kernel}: {tops:.1f} binary TOPS "
                  f"(2MNK / median), {tops / peak:.3f} of the measured tcgen05 kind::mxf4 peak "
                  f"({peak:.0f} TOPS)", file=err)
    csv_text = gemm.records_to_csv(records)
    if args.extended:
        lines = csv_text.rstrip("\n").split("\n")
        lines[0] += ",tops,roofline_frac"
        lines[1:] = [f"{ln},{t:.3f},{f:.4f}" for ln, (t, f) in zip(lines[1:], extra)]
        csv_text = "\n".join(lines) + "\n"
    print(csv_text, end="", file=out)
    if args.csv:
        tmp = args.csv + ".tmp"
        with open(tmp, "w") as f:
            f.write(csv_text)
        os.replace(tmp, args.csv)
    return EXIT_OK


def cmd_bench_gemm(args, **kw) -> int:
    from .gemm import GemmDims
    try:
        dims = GemmDims(args.M, args.N, args.K)
    except ValueError as exc:
        raise UsageError(str(exc)) from None
    return _run_bench([dims], args, **kw)


def cmd_bench_conv(args, **kw) -> int:
    from .gemm import GemmDims
    try:
        channels = [int(c) for c in args.channels.split(",") if c.strip()]
    except ValueError:
        raise UsageError(f"bad --channels list {args.channels!r}") from None
    if not channels:
        raise UsageError("no channel values given")
    n = args.batch * args.out_hw * args.out_hw
    try:
        dims_list = [GemmDims(args.filters, n, c * args.kernel_size * args.kernel_size)
                     for c in channels]
    except ValueError as exc:
        raise UsageError(str(exc)) from None
    return _run_bench(dims_list, args, **kw)


def main(argv=None) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
        return args.func(args)
    except UsageError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_USAGE
    except InternalCheckError as exc:
        print(f"internal error: {exc}", file=sys.stderr)
        return EXIT_INTERNAL
    except ValueError as exc:  # data errors (reference: IdxFormatError / ModelFormatError)
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_DATA

"""Bench CLI parity (``bitnn bench gemm|conv``, cli.py:139-156, 252-320): frozen CSV on
stdout, exit code 3 when the kernels' checksums disagree (cli.py:276-280), usage
errors exit 1.  The guard and the parsing run on CPU with a stubbed timer; the GPU
test runs every kernel id for real."""

import io

import numpy as np
import pytest

from paper_1705_09864_b200 import cli, gemm


def _fake(checksums):
    it = iter(checksums)

    def bench(kernel, dims, **kw):
        return gemm.BenchRecord(kernel=kernel, m=dims.m, n=dims.n, k=dims.k,
                                repeats=kw["repeats"], median_ns=1000, pack_ns=10,
                                checksum=next(it), seed=kw["seed"])
    return bench


def _run(monkeypatch, argv, checksums):
    monkeypatch.setattr(gemm, "benchmark_kernel", _fake(checksums))
    monkeypatch.setattr(cli, "mxf4_peak_tops", lambda: 8000.0)
    out, err = io.StringIO(), io.StringIO()
    args = cli.build_parser().parse_args(argv)
    return args.func(args, out=out, err=err), out.getvalue(), err.getvalue()


def test_frozen_csv_and_comments(monkeypatch):
    rc, out, err = _run(monkeypatch, ["bench", "gemm", "-M", "4", "-N", "5", "-K", "70",
                                      "--kernels", "xnor_base,xnor_b200", "--repeats", "3"],
                        [77, 77])
    assert rc == 0
    lines = out.strip().split("\n")
    assert lines[0] == "kernel,M,N,K,repeats,median_ns,pack_ns,checksum,seed"  # gemm.py:49
    assert lines[1] == "xnor_base,4,5,70,3,1000,10,77,0"
    assert lines[2].startswith("xnor_b200,4,5,70,3,")
    assert "binary TOPS" in err and "kind::mxf4" in err


def test_extended_columns(monkeypatch):
    rc, out, _ = _run(monkeypatch, ["bench", "gemm", "-M", "4", "-N", "5", "-K", "70",
                                    "--kernels", "xnor_b200", "--extended"], [1])
    assert rc == 0
    hdr, row = out.strip().split("\n")
    assert hdr.endswith(",tops,roofline_frac")
    tops = float(row.split(",")[-2])
    assert abs(tops - 2 * 4 * 5 * 70 / 1000 / 1e3) < 1e-3


def test_checksum_guard_exits_3(monkeypatch, capsys):
    monkeypatch.setattr(gemm, "benchmark_kernel", _fake([5, 6]))
    monkeypatch.setattr(cli, "mxf4_peak_tops", lambda: 8000.0)
    rc = cli.main(["bench", "gemm", "-M", "4", "-N", "5", "-K", "70", "--kernels",
                   "xnor_base,xnor_b200"])
    assert rc == cli.EXIT_INTERNAL == 3
    assert "disagree" in capsys.readouterr().err


def test_conv_sweep_dims(monkeypatch):
    rc, out, _ = _run(monkeypatch, ["bench", "conv", "--channels", "32,64", "--kernels",
                                    "xnor_parallel"], [1, 2])
    rows = [r.split(",") for r in out.strip().split("\n")[1:]]
    # cli.py:305-320: M = filters, N = batch * out_hw^2, K = C * k * k
    assert [(int(r[1]), int(r[2]), int(r[3])) for r in rows] == [(64, 200 * 64, 32 * 25),
                                                               (64, 200 * 64, 64 * 25)]


@pytest.mark.parametrize("argv", [
    ["bench", "gemm", "-M", "0", "-N", "5", "-K", "7"],
    ["bench", "gemm", "-M", "4", "-N", "5", "-K", "7", "--kernels", "nope"],
    ["bench", "gemm", "-M", "4", "-N", "5", "-K", "7", "--repeats", "0"],
    ["bench", "conv", "--channels", "a,b"],
    ["bench", "gemm", "-M", "100000", "-N", "100000", "-K", "100000"],
])
def test_usage_errors_exit_1(argv, capsys):
    assert cli.main(argv) == cli.EXIT_USAGE == 1
    assert "error:" in capsys.readouterr().err


@pytest.mark.gpu
def test_bench_gemm_all_kernels_on_gpu(tmp_path):
    """Every kernel id on the GPU: checksums agree (else exit 3), and equal the
    popcount-domain sum of the same seeded operands (make_operands), P = (dot + K) / 2
    (qmath.map_dot_to_xnor, pinned by test_gemm.py:17-34)."""
    csv = tmp_path / "r.csv"
    out, err = io.StringIO(), io.StringIO()
    args = cli.build_parser().parse_args(["bench", "gemm", "-M", "70", "-N", "90", "-K", "300",
                                          "--repeats", "2", "--csv", str(csv), "--seed", "4"])
    assert args.func(args, out=out, err=err) == 0
    assert csv.read_text() == out.getvalue()
    rows = [r.split(",") for r in out.getvalue().strip().split("\n")[1:]]
    assert [r[0] for r in rows] == list(gemm.KERNEL_IDS)
    a, b = gemm.make_operands(gemm.GemmDims(70, 90, 300), 4)
    p = (a.astype(np.float64) @ b.astype(np.float64) + 300) / 2
    assert {int(r[7]) for r in rows} == {int(round(float(p.sum())))}

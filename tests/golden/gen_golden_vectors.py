"""Generate golden vectors by running the UNMODIFIED reference (bitnn).

Run in the build container only (the reference is not on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/gen_golden_vectors.py

It imports the reference from /root/reference/pkg/src and writes small
fixtures next to this script.  Large outputs are stored as SHA-256 digests of
the reference's float32 output bytes (C order) plus a few sample values; the
inputs are regenerated from seeds by ``workloads.py`` wherever they are
needed.  Nothing under /root/reference is copied.
"""

from __future__ import annotations

import hashlib
import json
import os
import pathlib
import sys
import time

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
REF_SRC = os.environ.get("BITNN_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF_SRC)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from bitnn import bitpack, gemm, layers, qmath, tensor  # noqa: E402

import workloads as wl  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def gen_pack_cases(out):
    rng = np.random.default_rng(4)
    d = {}
    for i, (m, k) in enumerate(((1, 1), (5, 64), (7, 65), (32, 200), (3, 1000), (4, 70),
                                (2, 127), (9, 129))):
        x = rng.standard_normal((m, k)).astype(np.float32)
        x.reshape(-1)[::5] = 0.0
        x.reshape(-1)[2::9] = -0.0
        s = bitpack.binarize(x)
        d[f"x{i}"] = x
        d[f"signs{i}"] = s
        d[f"a{i}"] = bitpack.pack_matrix_a(s).words
        d[f"b{i}"] = bitpack.pack_matrix_b(np.ascontiguousarray(s.T)).words
    np.savez_compressed(out / "pack_cases.npz", **d)


def gen_gemm40(out):
    d = {}
    for i, (m, n, k, seed) in enumerate(wl.gemm40_cases()):
        a, b = wl.make_operands(m, n, k, seed)
        abm, bbm = bitpack.pack_matrix_a(a), bitpack.pack_matrix_b(b)
        c = gemm.xnor_gemm_base(abm, bbm)
        assert np.array_equal(c, qmath.map_dot_to_xnor(tensor.gemm_f32(a, b), k))
        d[f"a{i}"] = abm.words
        d[f"b{i}"] = bbm.words
        d[f"c{i}"] = c
        d[f"dims{i}"] = np.array([m, n, k], dtype=np.int64)
    np.savez_compressed(out / "gemm40.npz", **d)


def gen_sweep504(out):
    rows = []
    for m, n, k, a, b in wl.sweep504():
        c = gemm.xnor_gemm_parallel(bitpack.pack_matrix_a(a), bitpack.pack_matrix_b(b))
        rows.append([m, n, k, sha(c), int(c.astype(np.int64).sum())])
    (out / "sweep504.json").write_text(json.dumps(rows))


def gen_conv(out):
    d = {}
    for i, case in enumerate(wl.CONV_CASES):
        b, c, h, w, f, kh, kw, stride, pad, seed = case
        x, wt = wl.conv_case_inputs(case)
        # G2 composition of unmodified reference steps
        oh, ow = tensor.conv_output_hw(h, w, kh, kw, stride, pad)
        a_bm = bitpack.pack_matrix_a(bitpack.binarize(wt.reshape(f, -1)))
        cols = bitpack.binarize(tensor.im2col(x, kh, kw, stride, pad))
        y = gemm.xnor_gemm_base(a_bm, bitpack.pack_matrix_b(cols))
        y = y.reshape(f, b, oh, ow).transpose(1, 0, 2, 3)
        d[f"y{i}"] = np.ascontiguousarray(y)
        if pad == (0, 0):
            # the reference layer itself (QConv2d rejects padding, layers.py:178-180)
            layer = layers.QConv2d(c, f, (kh, kw), stride, (0, 0), bits=1)
            layer.weight = wt.copy()
            layer.pack()
            yl = layer.forward(bitpack.binarize(x), layers.INFER_PACKED)
            assert np.array_equal(yl, y)
    np.savez_compressed(out / "conv_cases.npz", **d)


def gen_layers(out):
    d = {}
    rng = np.random.default_rng(2)
    qd = layers.QDense(130, 17, bits=1, rng=rng)
    x = wl.random_signs(rng, (9, 130))
    d["qdense_w"] = qd.weight
    d["qdense_x"] = x
    d["qdense_y_float"] = qd.forward(x, layers.INFER_FLOAT)
    qd.pack()
    d["qdense_y_packed"] = qd.forward(x, layers.INFER_PACKED)
    d["qdense_words"] = qd.packed.words
    rng = np.random.default_rng(3)
    qc = layers.QConv2d(3, 5, (3, 3), bits=1, rng=rng)
    x = wl.random_signs(rng, (4, 3, 8, 8))
    d["qconv_w"] = qc.weight
    d["qconv_x"] = x
    d["qconv_y_float"] = qc.forward(x, layers.INFER_FLOAT)
    qc.pack()
    d["qconv_y_packed"] = qc.forward(x, layers.INFER_PACKED)
    d["qconv_words"] = qc.packed.words
    # QActivation on raw floats, incl. clipping and sign(0)
    xa = np.random.default_rng(5).standard_normal((6, 50)).astype(np.float32) * 2
    xa[0, :5] = [0.0, -0.0, 1.5, -1.5, 1e-30]
    d["qact_x"] = xa
    d["qact_y1"] = layers.QActivation(1).forward(xa, layers.INFER_PACKED)
    d["qact_y2"] = layers.QActivation(2).forward(xa, layers.INFER_FLOAT)
    np.savez_compressed(out / "layers.npz", **d)


def gen_qmath(out):
    rng = np.random.default_rng(21)
    x = rng.random((64, 96), dtype=np.float32)
    x.reshape(-1)[:8] = [0.0, 1.0, 1 / 6, 0.5, 5 / 6, 1 / 3, 2 / 3, 0.1666666716337204]
    xs = (rng.standard_normal((64, 96)) * 1.2).astype(np.float32)
    d = {"x": x, "q2": qmath.quantize(x, 2), "xs": xs, "qs2": qmath.quantize_signed(xs, 2),
         "qs1": qmath.quantize_signed(xs, 1)}
    # 2-bit dense: float64 oracle of the reference's float path (layers.py:370-377)
    w = rng.random((40, 96), dtype=np.float32)
    d["w"] = w
    d["dot2"] = qmath.quantize(x, 2).astype(np.float64) @ qmath.quantize(w, 2).astype(np.float64).T
    np.savez_compressed(out / "qmath.npz", **d)


def gen_configs(out):
    res = {}
    t0 = time.time()
    a, w = wl.config1_inputs()
    k = a.shape[1]
    p = gemm.xnor_gemm_parallel(bitpack.pack_matrix_a(bitpack.binarize(w)),
                                bitpack.pack_matrix_b(bitpack.binarize(np.ascontiguousarray(a.T))))
    y = np.ascontiguousarray(qmath.map_xnor_to_dot(p, k).T.astype(np.float32))  # [256, 1024]
    res["c1"] = {"sha256": sha(y), "sum": float(y.astype(np.float64).sum()),
                 "shape": list(y.shape), "sample": y[:2, :4].tolist(), "secs": time.time() - t0}
    t0 = time.time()
    x, wt = wl.config2_inputs()
    c = wl.C2
    oh, ow = tensor.conv_output_hw(c["h"], c["w"], c["kh"], c["kw"], c["stride"], c["pad"])
    a_bm = bitpack.pack_matrix_a(bitpack.binarize(wt.reshape(c["f"], -1)))
    cols = bitpack.binarize(tensor.im2col(x, c["kh"], c["kw"], c["stride"], c["pad"]))
    y = gemm.xnor_gemm_parallel(a_bm, bitpack.pack_matrix_b(cols))
    del cols
    y = np.ascontiguousarray(y.reshape(c["f"], c["b"], oh, ow).transpose(1, 0, 2, 3))
    res["c2"] = {"sha256": sha(y), "sum": float(y.astype(np.float64).sum()),
                 "shape": list(y.shape), "sample": y[0, 0, 0, :4].tolist(),
                 "secs": time.time() - t0}
    (out / "configs.json").write_text(json.dumps(res, indent=1))


def gen_bmx(out):
    """Golden .bmx files written by the reference's own modelio (test_modelio.py:37-45)."""
    sys.path.insert(0, os.path.join(os.path.dirname(REF_SRC), "tests", "data"))
    import gen_golden  # the reference's fixture builder, imported (not copied)
    from bitnn import modelio
    net = gen_golden.build_golden_net()
    fp, pp = out / "golden_float.bmx", out / "golden_packed.bmx"
    modelio.save_model(net, fp)
    modelio.convert(fp, pp)
    x = gen_golden.probe_input()
    probs_f = modelio.load_model(fp).forward(x, layers.INFER_FLOAT)
    probs_p = modelio.load_model(pp).forward(x, layers.INFER_PACKED)
    meta = {"float_sha256": hashlib.sha256(fp.read_bytes()).hexdigest(),
            "packed_sha256": hashlib.sha256(pp.read_bytes()).hexdigest(),
            "float_size": fp.stat().st_size, "packed_size": pp.stat().st_size,
            "probe_seed": gen_golden.SEED + 1, "probs_float": probs_f.tolist(),
            "probs_packed": probs_p.tolist()}
    (out / "golden_bmx.json").write_text(json.dumps(meta, indent=1))


def gen_lenet_bmx(out):
    """The reference's own binary LeNet (layers.build_lenet(binary=True): kernel given as a
    (5, 5) tuple, MaxPool2d(), QDense 1024 -> 1000) written by its modelio and converted to
    packed weights; probe probabilities of both modes from the reference's forward."""
    from bitnn import modelio
    net = layers.build_lenet(binary=True, seed=0)
    # BatchNorm running statistics calibrated on a separate batch (the reference's own
    # train-mode statistics): an untrained net with unit statistics saturates its tanh
    # and maps every image to the same output
    rng = np.random.default_rng(11)
    t = (rng.standard_normal((64, 1, 28, 28)) * 2).astype(np.float32)
    for layer in net.layers:
        if isinstance(layer, layers.BatchNorm):
            c = layer.channels
            axes = (0, 2, 3) if t.ndim == 4 else (0,)
            layer.gamma = (0.5 + rng.random(c)).astype(np.float32)
            layer.beta = (rng.standard_normal(c) * 0.1).astype(np.float32)
            layer.running_mean = t.mean(axis=axes).astype(np.float32)
            layer.running_var = (t.var(axis=axes) + 1.0).astype(np.float32)
        t = layer.forward(t, layers.INFER_FLOAT)
    fp, pp = out / "_lenet_float.bmx", out / "lenet_packed.bmx"
    modelio.save_model(net, fp)
    modelio.convert(fp, pp)
    fp.unlink()
    x = (np.random.default_rng(7).standard_normal((4, 1, 28, 28)) * 2).astype(np.float32)
    packed = modelio.load_model(pp)
    meta = {"packed_sha256": hashlib.sha256(pp.read_bytes()).hexdigest(),
            "probe_seed": 7, "probe_shape": [4, 1, 28, 28],
            "probs_packed": packed.forward(x, layers.INFER_PACKED).tolist(),
            "probs_float_of_seed0": net.forward(x, layers.INFER_FLOAT).tolist()}
    (out / "lenet_bmx.json").write_text(json.dumps(meta, indent=1))


def main():
    out = HERE
    only = set(sys.argv[1:])  # optional: names of the generators to run
    for fn in (gen_pack_cases, gen_gemm40, gen_conv, gen_layers, gen_qmath, gen_sweep504,
               gen_configs, gen_bmx, gen_lenet_bmx):
        if only and fn.__name__ not in only:
            continue
        t0 = time.time()
        fn(out)
        print(f"{fn.__name__}: {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main()

"""``.bmx`` loader against golden files written by the reference.

tests/golden/golden_{float,packed}.bmx were produced by the reference's own
writer (gen_golden_vectors.py -> bitnn.modelio.save_model / convert); their
SHA-256 match the reference's pinned digests (test_modelio.py:37-45).
"""

import hashlib
import json
import os

import numpy as np
import pytest
import torch

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _meta():
    return json.load(open(os.path.join(GOLD, "golden_bmx.json")))


def test_golden_files_are_the_reference_bytes():
    meta = _meta()
    for kind in ("float", "packed"):
        data = open(os.path.join(GOLD, f"golden_{kind}.bmx"), "rb").read()
        assert len(data) == meta[f"{kind}_size"]
        assert hashlib.sha256(data).hexdigest() == meta[f"{kind}_sha256"]
    assert meta["float_sha256"].startswith("03066a60") and meta["packed_sha256"].startswith("71f23e6c")


def test_format_errors_cpu(tmp_path):
    from paper_1705_09864_b200.modelio import ModelFormatError, load_model
    good = open(os.path.join(GOLD, "golden_packed.bmx"), "rb").read()
    for bad, msg in ((b"XMX1" + good[4:], "bad magic"), (good[:4] + b"\x02\x00\x00\x00" + good[8:],
                                                        "unsupported version"),
                     (good[:10], "truncated")):
        p = tmp_path / "bad.bmx"
        p.write_bytes(bad)
        with pytest.raises(ModelFormatError, match=msg):
            load_model(p)


@pytest.mark.gpu
def test_packed_golden_probe_probs():
    import paper_1705_09864_b200 as bnn
    from paper_1705_09864_b200.modelio import load_model
    meta = _meta()
    net = load_model(os.path.join(GOLD, "golden_packed.bmx"))
    x = np.random.default_rng(meta["probe_seed"]).standard_normal((2, 1, 12, 12)).astype(np.float32)
    probs = net.forward(x, bnn.INFER_PACKED)
    assert np.allclose(probs, np.array(meta["probs_packed"]), atol=1e-6, rtol=0)


@pytest.mark.gpu
def test_float_and_packed_files_agree_at_binary_layers():
    import paper_1705_09864_b200 as bnn
    from paper_1705_09864_b200.modelio import load_model
    fnet = load_model(os.path.join(GOLD, "golden_float.bmx"))
    pnet = load_model(os.path.join(GOLD, "golden_packed.bmx"))
    for l in fnet.quantized_layers:
        l.pack()  # convert in place, as modelio.convert does
    x = np.random.default_rng(0).standard_normal((16, 1, 12, 12)).astype(np.float32)
    cf, cp = [], []
    pf = fnet.forward(x, bnn.INFER_FLOAT, capture=cf)
    pp = pnet.forward(x, bnn.INFER_PACKED, capture=cp)
    for i, layer in enumerate(fnet.layers):
        if isinstance(layer, (bnn.QConv2d, bnn.QDense)):
            assert np.array_equal(cf[i], cp[i]), i
    assert np.allclose(pf, pp, atol=1e-5, rtol=0)  # verify_equivalence (modelio.py:299-324)
    # packed words from the file == words packed on the GPU from the float masters
    for a, b in zip(fnet.quantized_layers, pnet.quantized_layers):
        assert torch.equal(a.packed.words, b.packed.words)


def test_flipped_tail_bit_is_rejected(tmp_path):
    """A set tail bit in a packed payload fails the padding audit (test_modelio.py:381-393)."""
    from paper_1705_09864_b200.modelio import ModelFormatError, load_model
    data = bytearray(open(os.path.join(GOLD, "golden_packed.bmx"), "rb").read())
    # the last tensor payloads are float; find the qconv payload: K = 4*3*3 = 36 bits -> tail bits 36..63
    name = b"layer5.weight"
    i = data.index(name) + len(name) + 2 + 8 * 2  # dtype, ndim, 2 dims
    data[i + 7] |= 0x80  # bit 63 of the first word
    p = tmp_path / "flip.bmx"
    p.write_bytes(bytes(data))
    with pytest.raises(ModelFormatError, match="padding audit"):
        load_model(p)


def test_reference_lenet_file_is_the_reference_bytes():
    meta = json.load(open(os.path.join(GOLD, "lenet_bmx.json")))
    data = open(os.path.join(GOLD, "lenet_packed.bmx"), "rb").read()
    assert hashlib.sha256(data).hexdigest() == meta["packed_sha256"]


def test_conv2d_accepts_pairs_like_the_reference():
    """Reference Conv2d takes (kh, kw) / (sh, sw) / (ph, pw) tuples (layers.py:86-141);
    the .bmx reader installs them as read (tuples), the builders as ints."""
    from paper_1705_09864_b200 import nets
    c = nets.Conv2d(3, 8, (5, 3), stride=(2, 1), pad=(2, 0), bias=False)
    assert c.weight.shape == (8, 3, 5, 3)
    assert c.geometry() == (5, 3, 2, 1, 2, 0)
    assert c.output_hw(28, 28) == (14, 26)
    c.stride, c.pad = (1, 1), (0, 0)  # as modelio._Conv2d re-assigns them
    assert c.output_hw(28, 28) == (24, 26)
    assert nets.Conv2d(1, 64, 5, pad=2).geometry() == (5, 5, 1, 1, 2, 2)


@pytest.mark.gpu
def test_reference_lenet_round_trip_forward():
    """The reference's own build_lenet(binary=True) -- conv kernel given as a (5, 5) tuple,
    64 filters, so the tensor-core stem engine runs -- saved and converted by the
    reference's modelio, loaded here and run in infer_packed mode: probabilities equal to
    the reference's forward of the same file (float stem / BN / tanh rounding only)."""
    import paper_1705_09864_b200 as bnn
    from paper_1705_09864_b200.modelio import load_model
    meta = json.load(open(os.path.join(GOLD, "lenet_bmx.json")))
    net = load_model(os.path.join(GOLD, "lenet_packed.bmx"))
    conv = net.layers[0]
    assert conv.tc_supported() and conv.geometry() == (5, 5, 1, 1, 0, 0)
    x = (np.random.default_rng(meta["probe_seed"]).standard_normal(meta["probe_shape"])
         * 2).astype(np.float32)
    want = np.array(meta["probs_packed"])
    probs = net.forward(x, bnn.INFER_PACKED)
    assert probs.shape == want.shape
    assert np.array_equal(probs.argmax(1), want.argmax(1))
    assert np.allclose(probs, want, atol=2e-5, rtol=0)
    conv.engine = "cudnn"  # the other float engine agrees as well
    assert np.allclose(net.forward(x, bnn.INFER_PACKED), want, atol=2e-5, rtol=0)

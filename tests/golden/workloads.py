"""Seeded synthetic workloads shared by the golden generator, tests and bench.

Everything here is deterministic NumPy (PCG64 via ``np.random.default_rng``)
so the GPU box regenerates bit-identical inputs from a seed instead of
shipping large fixtures.  The case lists replay the generation procedure of
the reference's own tests (``pkg/tests/test_gemm.py:17-34`` and
``pkg/tests/test_acceptance.py:99-127``) so that the golden hashes computed
by the reference in this container can be checked on the GPU box.
"""

from __future__ import annotations

import numpy as np

# BASELINE.json configs: seeds are fixed and recorded here.
C1 = dict(name="qfc_1024x256x4096", batch=256, units=1024, k=4096, seed=1)
C2 = dict(name="qconv3x3_256_32x28x28", b=32, c=256, h=28, w=28, f=256, kh=3, kw=3,
          stride=(1, 1), pad=(1, 1), seed=2)
C5_SQUARE = (4096, 8192, 16384)
C5_LONGK = (4096, 4096, 65536)


def make_operands(m: int, n: int, k: int, seed: int):
    """gemm.make_operands (gemm.py:354-360): +-1 float32 A [m,k], B [k,n]."""
    rng = np.random.default_rng(seed)
    choices = np.array([-1.0, 1.0], dtype=np.float32)
    a = rng.choice(choices, size=(m, k))
    b = rng.choice(choices, size=(k, n))
    return a, b


def random_signs(rng, shape):
    """conftest.random_signs / test_acceptance._random_signs."""
    return np.where(rng.random(shape) < 0.5, -1.0, 1.0).astype(np.float32)


def gemm40_cases():
    """The 40 (m, n, k) shapes and operand seeds of test_gemm.py:17-34."""
    rng = np.random.default_rng(0)
    cases = [(1, 1, 1), (1, 1, 63), (1, 1, 64), (1, 1, 65), (2, 3, 128)]
    while len(cases) < 40:
        cases.append((int(rng.integers(1, 64)), int(rng.integers(1, 64)),
                      int(rng.integers(1, 1024))))
    return [(m, n, k, len(cases) + m + n + k) for m, n, k in cases]


def sweep504():
    """Yield (m, n, k, a, b) in the exact rng order of test_acceptance.py:99-127."""
    rng = np.random.default_rng(1001)
    triples = [(1, 1, k) for k in (1, 63, 64, 65)]
    while len(triples) < 504:
        triples.append((int(rng.integers(1, 129)), int(rng.integers(1, 129)),
                        int(rng.integers(1, 4097))))
    for m, n, k in triples:
        a = random_signs(rng, (m, k))
        b = random_signs(rng, (k, n))
        yield m, n, k, a, b


def config1_inputs(seed: int = C1["seed"]):
    """C1: A (activations) U[-1,1] [256, 4096]; W U[-1,1] [1024, 4096] (float32)."""
    rng = np.random.default_rng(seed)
    a = rng.uniform(-1.0, 1.0, size=(C1["batch"], C1["k"])).astype(np.float32)
    w = rng.uniform(-1.0, 1.0, size=(C1["units"], C1["k"])).astype(np.float32)
    return a, w


def config2_inputs(seed: int = C2["seed"]):
    """C2: x N(0,1) [32,256,28,28]; W N(0,1) [256,256,3,3] (float32)."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((C2["b"], C2["c"], C2["h"], C2["w"]), dtype=np.float32)
    w = rng.standard_normal((C2["f"], C2["c"], C2["kh"], C2["kw"]), dtype=np.float32)
    return x, w


CONV_CASES = [
    # (B, C, H, W, F, kh, kw, stride, pad, seed) -- small, ragged channel counts
    (2, 3, 7, 6, 4, 3, 3, (1, 1), (0, 0), 11),
    (2, 3, 7, 6, 4, 3, 3, (1, 1), (1, 1), 12),
    (1, 5, 9, 8, 3, 3, 3, (2, 1), (1, 0), 13),
    (3, 64, 6, 6, 5, 5, 5, (1, 1), (2, 2), 14),
    (2, 70, 5, 7, 6, 3, 3, (2, 2), (2, 1), 15),
    (1, 130, 4, 4, 7, 1, 1, (1, 1), (0, 0), 16),
    (2, 32, 8, 8, 9, 3, 3, (1, 1), (1, 1), 17),
    (1, 128, 5, 5, 8, 2, 2, (1, 1), (0, 0), 18),
]


def conv_case_inputs(case):
    b, c, h, w, f, kh, kw, stride, pad, seed = case
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((b, c, h, w), dtype=np.float32)
    # a few exact zeros and negative zeros: sign(0) = sign(-0) = +1
    flat = x.reshape(-1)
    flat[:: 7] = 0.0
    flat[3:: 11] = -0.0
    wt = rng.standard_normal((f, c, kh, kw), dtype=np.float32)
    return x, wt

"""World-size-2 gloo tests of the N-split GEMM host logic (CPU only).

The GPU kernel is replaced by the pinned CPU oracle through the injectable
``compute`` hook, so partitioning, shard padding and all-gather order are
checked exactly like the reference's worker-count determinism test
(test_gemm.py:52-59): the gathered output must equal the single-process
result bit for bit.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1705_09864_b200.parallel import NsplitGemm, batch_shard, nsplit_xnor_gemm, shard_bounds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_compute(a_rows, b_rows, k, out):
    from oracle import oracle as orc
    x = orc.xor_popc_rowrow(b_rows.numpy().view(np.uint64), a_rows.numpy().view(np.uint64))
    out.copy_(torch.from_numpy((k - x).astype(np.float32)))


def _worker(rank, world, port, m, n, k, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(seed)
        w = (k + 63) // 64
        a = torch.randint(-2**62, 2**62, (m, w), generator=g)
        b = torch.randint(-2**62, 2**62, (n, w), generator=g)
        if k % 64:
            a[:, -1] &= (1 << (k % 64)) - 1
            b[:, -1] &= (1 << (k % 64)) - 1
        c = nsplit_xnor_gemm(a, b, k, compute=_oracle_compute)
        n0, n1, _ = shard_bounds(n, world, rank)
        plan = NsplitGemm(a, b[n0:n1], k, n, compute=_oracle_compute)  # the bench's step
        c2 = plan.run()
        assert torch.equal(c, c2)
        q.put((rank, c.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m,n,k", [(8, 13, 130), (5, 2, 64), (16, 31, 1000), (3, 1, 70)])
def test_nsplit_matches_single_process(m, n, k):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if root not in sys.path:
        sys.path.insert(0, root)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, n, k, 7, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process reference of the same operands
    g = torch.Generator().manual_seed(7)
    w = (k + 63) // 64
    a = torch.randint(-2**62, 2**62, (m, w), generator=g)
    b = torch.randint(-2**62, 2**62, (n, w), generator=g)
    if k % 64:
        a[:, -1] &= (1 << (k % 64)) - 1
        b[:, -1] &= (1 << (k % 64)) - 1
    single = torch.zeros((n, m))
    _oracle_compute(a, b, k, single)
    for r in range(world):
        assert results[r].shape == (n, m)
        assert np.array_equal(results[r], single.numpy()), f"rank {r}"


def test_shard_bounds_partition():
    for n in (0, 1, 7, 8, 9, 100):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(n, world, r) for r in range(world)]
            covered = [i for n0, n1, _ in spans for i in range(n0, n1)]
            assert covered == list(range(n))
            assert len({s for _, _, s in spans}) == 1
    assert batch_shard(256, 8, 7) == (224, 256)
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def test_bench_self_launch_command(monkeypatch):
    """``bench.py --gpus N`` without WORLD_SIZE re-launches itself as N ranks through
    torch.distributed.run on 127.0.0.1 (the driver's own launch line)."""
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import bench
    seen = {}
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: seen.setdefault("cmd", cmd) and 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "3"])
    args = bench.parse()
    assert args.workload == "resnet18" and args.gpus == 4
    bench.spawn_ranks(args)
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "3"]
    assert bench.SCALING["resnet18"] == "strong" and bench.SCALING["c2"] == "weak"

"""World-size-2 runs of the sharded paths with the REAL CUDA kernels.

Two ``gloo`` ranks share cuda:0: each runs its own shard through libbnn_b200 and
the shards are gathered through host memory (parallel.all_gather_rows).  No kernel
waits on another rank (the only cross-rank step is the host-side gloo gather), so
running both ranks on one device is safe.  The gathered results must equal the
one-process results bit for bit, like the reference's worker-count determinism
(test_gemm.py:52-59):
* the N-split config-5 GEMM (each rank an N shard, all-gather of [N/g, M] shards);
* batch-sharded ResNet-18 inference (each rank a batch shard, logits gathered).
"""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gemm_operands(m, n, k, seed):
    g = torch.Generator().manual_seed(seed)
    w = (k + 63) // 64
    a = torch.randint(-2**62, 2**62, (m, w), generator=g)
    b = torch.randint(-2**62, 2**62, (n, w), generator=g)
    if k % 64:
        a[:, -1] &= (1 << (k % 64)) - 1
        b[:, -1] &= (1 << (k % 64)) - 1
    return a.view(torch.uint64), b.view(torch.uint64)


def _worker(rank, world, port, what, q):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_1705_09864_b200 as bnn
        from paper_1705_09864_b200.parallel import (NsplitGemm, all_gather_rows,
                                                    nsplit_xnor_gemm, shard_bounds)
        bnn.load_library()
        if what == "gemm":
            out = {}
            for m, n, k in ((300, 1000, 4096), (256, 25088 // 8, 2304), (70, 129, 1000)):
                a, b = _gemm_operands(m, n, k, m + n + k)
                a, b = a.cuda(), b.cuda()
                c = nsplit_xnor_gemm(a, b, k)
                n0, n1, _ = shard_bounds(n, world, rank)
                plan = NsplitGemm(a, b[n0:n1].contiguous(), k, n)
                c2 = plan.run()
                torch.cuda.synchronize()
                out[(m, n, k)] = (c.cpu().numpy(), c2.cpu().numpy())
            q.put((rank, out))
        else:
            from paper_1705_09864_b200 import nets
            net = nets.resnet18_c4(seed=6)
            net.pack_for_inference()
            x = torch.randn((6, 3, 224, 224), generator=torch.Generator().manual_seed(8))
            b0, b1, shard = shard_bounds(6, world, rank)
            y = net.forward(x[b0:b1].cuda(), bnn.INFER_PACKED)
            local = torch.zeros((shard, y.shape[1]), dtype=torch.float32, device="cuda")
            local[: b1 - b0] = y
            full = torch.empty((shard * world, y.shape[1]), dtype=torch.float32, device="cuda")
            all_gather_rows(full, local)
            q.put((rank, full[:6].cpu().numpy()))
    finally:
        dist.destroy_process_group()


def _run(what, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, what, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return results


def test_nsplit_gemm_two_ranks_real_kernel():
    import paper_1705_09864_b200 as bnn
    results = _run("gemm")
    bnn.load_library()
    for (m, n, k) in results[0]:
        a, b = _gemm_operands(m, n, k, m + n + k)
        single = bnn.xnor_rows_gemm(a.cuda(), b.cuda(), k, transpose_out=True).cpu().numpy()
        for r in results:
            got, got_plan = results[r][(m, n, k)]
            assert got.shape == (n, m)
            assert np.array_equal(got, single), (r, m, n, k)
            assert np.array_equal(got_plan, single), (r, m, n, k)


def test_batch_sharded_resnet18_two_ranks_real_kernels():
    import paper_1705_09864_b200 as bnn
    from paper_1705_09864_b200 import nets
    results = _run("resnet")
    net = nets.resnet18_c4(seed=6)
    net.pack_for_inference()
    x = torch.randn((6, 3, 224, 224), generator=torch.Generator().manual_seed(8))
    single = net.forward(x.cuda(), bnn.INFER_PACKED).cpu().numpy()
    for r in results:
        assert np.array_equal(results[r], single), r

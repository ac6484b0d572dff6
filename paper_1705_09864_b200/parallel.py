"""Multi-GPU sharding of the binary GEMM and of whole-network inference.

Large GEMMs (config 5) split along N (activation rows): every rank keeps the
full packed weights A [M, W], computes the output shard C[n0:n1, :] for its
contiguous slice of B, and the shards are gathered with one
``all_gather_into_tensor`` (NCCL over NVLink on the B200 box).  Output is
N-major ([N, M]) so each shard is one contiguous block and the gather is a
pure copy -- results are bit-identical for any world size, the GPU analogue of
the reference's disjoint row partition (xnor_gemm_parallel, gemm.py:254-284;
test_gemm.py:52-59).

Whole-network inference shards the batch (``batch_shard``) with no collective
on the data path: every image's output is computed by exactly one rank with
per-image kernels, so the union of the shards equals the one-GPU result.

With a ``gloo`` process group (the CPU tests, or several ranks sharing one
device) the gather is staged through host memory; with ``nccl`` it runs on the
device.  The compute callable is injectable so the host-side logic (partition,
padding to equal shards, gather order) is also testable without a GPU.
"""

from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int, int]:
    """Contiguous balanced split: (n0, n1, shard) with shard = ceil(n / world).

    Ranks past the end get empty ranges; every rank's buffer is ``shard``
    rows so ``all_gather_into_tensor`` sees equal sizes.
    """
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    shard = (n + world - 1) // world
    n0 = min(n, rank * shard)
    n1 = min(n, n0 + shard)
    return n0, n1, shard


def _world(group):
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


def all_gather_rows(full: torch.Tensor, local: torch.Tensor, group=None) -> torch.Tensor:
    """``full`` [world * shard, ...] <- every rank's ``local`` [shard, ...], rank order.

    NCCL gathers device tensors in place; gloo (host backend) gathers through
    pinned host staging and copies back, so the same call works on either."""
    if dist.get_backend(group) == "nccl" or not local.is_cuda:
        dist.all_gather_into_tensor(full, local, group=group)
        return full
    host_full = torch.empty(full.shape, dtype=full.dtype)
    dist.all_gather_into_tensor(host_full, local.cpu(), group=group)
    full.copy_(host_full)
    return full


def _default_compute(a_rows, b_rows, k, out):
    from .gemm import xnor_rows_gemm
    return xnor_rows_gemm(a_rows, b_rows, k, out=out, transpose_out=True)


def nsplit_xnor_gemm(a_rows: torch.Tensor, b_rows: torch.Tensor, k: int, *,
                     group=None, compute: Callable | None = None,
                     out: torch.Tensor | None = None) -> torch.Tensor:
    """N-sharded xnor GEMM with one all-gather.

    ``a_rows`` [M, W]: full packed weights on every rank.  ``b_rows`` [N, W]:
    the full packed activations (each rank reads only its slice).
    Returns the popcount-domain output [N, M] on every rank.
    """
    world, rank = _world(group)
    compute = compute or _default_compute
    m, n = a_rows.shape[0], b_rows.shape[0]
    n0, n1, shard = shard_bounds(n, world, rank)
    local = torch.zeros((shard, m), dtype=torch.float32, device=a_rows.device)
    if n1 > n0:
        compute(a_rows, b_rows[n0:n1], k, local[: n1 - n0])
    if world == 1:
        if out is not None:
            out.copy_(local[:n])
            return out
        return local[:n]
    full = torch.empty((shard * world, m), dtype=torch.float32, device=a_rows.device)
    all_gather_rows(full, local, group)
    result = full[:n]
    if out is not None:
        out.copy_(result)
        return out
    return result


class NsplitGemm:
    """Pre-allocated N-split GEMM step (bench / serving): this rank's B shard, its
    [shard, M] output and the gathered [world * shard, M] result.  ``compute()`` is
    one kernel launch (no collective, CUDA-graph capturable); ``gather()`` is the
    collective; ``run()`` both."""

    def __init__(self, a_rows: torch.Tensor, b_rows_shard: torch.Tensor, k: int, n_total: int,
                 group=None, algo="auto", compute: Callable | None = None):
        self.world, self.rank = _world(group)
        self.group = group
        self.a, self.k, self.n = a_rows, k, n_total
        # ([rows, W] words, or [bits, rows, W] bit planes of the multi-bit path)
        self.m = a_rows.shape[-2]
        self.n0, self.n1, self.shard = shard_bounds(n_total, self.world, self.rank)
        if b_rows_shard.shape[-2] != self.n1 - self.n0:
            raise ValueError(f"rank {self.rank} expects {self.n1 - self.n0} rows of B, "
                             f"got {b_rows_shard.shape[-2]}")
        self.b = b_rows_shard
        self.algo = algo
        self._compute = compute
        self.local = torch.zeros((self.shard, self.m), dtype=torch.float32, device=a_rows.device)
        self.full = torch.empty((self.shard * self.world, self.m), dtype=torch.float32,
                                device=a_rows.device)

    def compute(self):
        if self.n1 > self.n0:
            if self._compute is not None:
                self._compute(self.a, self.b, self.k, self.local[: self.n1 - self.n0])
            else:
                from .gemm import xnor_rows_gemm
                xnor_rows_gemm(self.a, self.b, self.k, out=self.local[: self.n1 - self.n0],
                               transpose_out=True, algo=self.algo)
        return self.local

    def gather(self):
        if self.world == 1:
            self.full.copy_(self.local)
        else:
            all_gather_rows(self.full, self.local, self.group)
        return self.full[: self.n]

    def run(self):
        self.compute()
        return self.gather()


def batch_shard(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Replica partition of a batch for whole-network inference (no collective)."""
    b0, b1, _ = shard_bounds(batch, world, rank)
    return b0, b1

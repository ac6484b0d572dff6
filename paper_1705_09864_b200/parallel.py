"""Multi-GPU sharding of the binary GEMM.

Large GEMMs (config 5) split along N (activation rows): every rank keeps the
full packed weights A [M, W], computes the output shard C[n0:n1, :] for its
contiguous slice of B, and the shards are gathered with one
``all_gather_into_tensor`` (NCCL over NVLink on the B200 box).  Output is
N-major ([N, M]) so each shard is one contiguous block and the gather is a
pure copy -- results are bit-identical for any world size, the GPU analogue of
the reference's disjoint row partition (xnor_gemm_parallel, gemm.py:254-284;
test_gemm.py:52-59).

Whole-network inference shards by batch with no collective (replicas).

The compute callable is injectable so the host-side logic (partition,
padding to equal shards, gather order) is testable on CPU with gloo.
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


def _default_compute(a_rows, b_rows, k, out):
    from .gemm import xnor_rows_gemm
    return xnor_rows_gemm(a_rows, b_rows, k, out=out, transpose_out=True)


def nsplit_xnor_gemm(a_rows: torch.Tensor, b_rows: torch.Tensor, k: int, *,
                     group=None, compute: Callable | None = None,
                     out: torch.Tensor | None = None) -> torch.Tensor:
    """N-sharded xnor GEMM with one all-gather.

    ``a_rows`` [M, W]: full packed weights on every rank.  ``b_rows`` [N, W]:
    the full packed activations (each rank reads only its slice) .
    Returns the popcount-domain output [N, M] on every rank.
    """
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
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
    dist.all_gather_into_tensor(full, local, group=group)
    result = full[:n]
    if out is not None:
        out.copy_(result)
        return out
    return result


def batch_shard(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Replica partition of a batch for whole-network inference (no collective)."""
    b0, b1, _ = shard_bounds(batch, world, rank)
    return b0, b1

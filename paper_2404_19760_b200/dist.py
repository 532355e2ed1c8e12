"""Data parallelism over rays.

Rays are independent in both passes ("each kernel instance is
responsible for a single ray"), so a batch shards over ranks with no exchange
in the forward or the backward march. The one real exchange (row X1) is the sum
of the theta and MLP gradients across ranks: one in-place all-reduce of a flat
fp32 buffer [grad planes | grad params] (NCCL over NVLink/NVSwitch on GPUs,
gloo in the CPU tests).
"""
from __future__ import annotations

from typing import Callable, List, Sequence, Tuple

import torch
import torch.distributed as dist


def shard_range(n_total: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous ray range [lo, hi) of `rank`; sizes differ by at most one ray."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    return rank * n_total // world, (rank + 1) * n_total // world


class FlatGrads:
    """One flat buffer holding every gradient tensor, each piece 16-byte aligned
    (the C ABI's vector reductions need it), so the cross-rank reduction is a
    single collective with no pack/unpack kernels."""

    def __init__(self, shapes: Sequence[Sequence[int]], device=None, dtype=torch.float32):
        self.shapes = [tuple(int(x) for x in s) for s in shapes]
        sizes = [int(torch.Size(s).numel()) for s in self.shapes]
        align = 16 // torch.tensor([], dtype=dtype).element_size()
        offs, o = [], 0
        for n in sizes:
            offs.append(o)
            o += (n + align - 1) // align * align
        self.flat = torch.zeros(o, device=device, dtype=dtype)
        self.views: List[torch.Tensor] = [self.flat[a:a + n].view(s) for a, n, s in zip(offs, sizes, self.shapes)]

    def zero_(self):
        self.flat.zero_()
        return self


def allreduce_grads(grads: FlatGrads, group=None) -> FlatGrads:
    """Sum the gradient buffer over all ranks in place (no-op when not distributed)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(grads.flat, op=dist.ReduceOp.SUM, group=group)
    return grads


def dp_backward(n_total: int, backward_shard: Callable[[int, int, List[torch.Tensor]], None], grads: FlatGrads,
                group=None) -> FlatGrads:
    """One data-parallel backward: this rank accumulates the gradients of its ray
    shard into `grads` (backward_shard(lo, hi, views)), then the buffer is summed
    across ranks. With the CUDA path, backward_shard calls lp_render_backward."""
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    lo, hi = shard_range(n_total, rank, world)
    if hi > lo:
        backward_shard(lo, hi, grads.views)
    return allreduce_grads(grads, group)

"""Multi-GPU sharding of the hot path (one process per GPU, torch.distributed
over NCCL for the one real exchange step).

Rasterizer: views are independent (rasterizer.cpp:112-342 is a function of one
angle). Rank r renders views r, r+N, ... of the batch into its local per-kernel
gradients; one all-reduce (sum) of the 11*M gradient buffer (+ the adaptive
statistics when requested) completes the step. Every rank then holds the
gradients the reference gets by calling render_backward once per view into one
CloudGrads (accumulate semantics, rasterizer.cpp:329-331).

Voxelizer: per-brick lists are independent (voxelizer.cpp:115-136), so ranks
take contiguous z-slabs of 8-voxel brick layers; each writes its slab of the
volume, and the per-kernel partial gradients of voxelize_backward are
all-reduced. Slab boundaries balance the (brick, kernel) pair counts when a
per-layer weight is given.
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple


def shard_views(n_views: int, rank: int, world: int) -> List[int]:
    """Strided view assignment: rank r gets r, r+world, ... (max-min <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return list(range(rank, n_views, world))


def shard_z_bricks(n_layers: int, rank: int, world: int,
                   weights: Optional[Sequence[float]] = None) -> Tuple[int, int]:
    """Contiguous [z0, z1) range of brick layers for `rank`. Without weights
    the layers are split evenly; with per-layer weights (e.g. pair counts)
    the cumulative weight is split evenly. The ranges of all ranks partition
    [0, n_layers)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if weights is None:
        base, extra = divmod(n_layers, world)
        z0 = rank * base + min(rank, extra)
        return z0, z0 + base + (1 if rank < extra else 0)
    assert len(weights) == n_layers
    total = float(sum(weights))
    if total <= 0.0:
        return shard_z_bricks(n_layers, rank, world)
    cuts = [0]
    acc, k = 0.0, 1
    for z, w in enumerate(weights):
        acc += w
        while k < world and acc >= total * k / world:
            cuts.append(z + 1)
            k += 1
    while len(cuts) < world:
        cuts.append(n_layers)
    cuts.append(n_layers)
    return cuts[rank], cuts[rank + 1]


def allreduce_(tensors, group=None):
    """Sum-all-reduce each tensor in place (NCCL on CUDA tensors, gloo on CPU)."""
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    for t in tensors:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)


def allreduce_grads(grads, cloud=None, group=None):
    """One collective for the whole 11*M gradient buffer (CloudGrads.buffer);
    plus the adaptive statistics of `cloud` when given."""
    allreduce_([grads.buffer], group)
    if cloud is not None:
        allreduce_([cloud.grad2d_norm_accum, cloud.grad_count, cloud.grad3d_accum], group)

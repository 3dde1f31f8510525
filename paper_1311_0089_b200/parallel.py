"""Multi-GPU plumbing for the slab-decomposed solver.

One process per GPU (torchrun).  torch.distributed carries only the host-side
plumbing: the NCCL unique id of the library's communicator (broadcast from
rank 0), the max-over-ranks timing, and assembling slab results on rank 0.
The data path (two axis-0 exchanges per operator application, the CG / fixed-
point reductions) runs inside the CUDA library over NCCL (fc_create_dist).

The partitions mirror the library exactly (fc_engine.cu::create_slab):
slab t owns axis-0 planes [t n0 / P, (t+1) n0 / P) and outer pencils
[t Q / P, (t+1) Q / P), Q = n1 (n2 + 1) / 2.
"""

from __future__ import annotations

import numpy as np


def slab_bounds(n0: int, P: int):
    """Axis-0 plane ranges per slab (uneven: 729 / 8 -> 91 or 92 planes)."""
    return [(t * n0 // P, (t + 1) * n0 // P) for t in range(P)]


def pencil_bounds(shape, P: int):
    """Outer-sweep (k2, k1) pencil ranges per slab for a 3-D grid."""
    Q = shape[1] * ((shape[2] + 1) // 2)
    return [(t * Q // P, (t + 1) * Q // P) for t in range(P)]


def exchange_counts(shape, R: int, P: int):
    """Complex elements slab s sends to slab p in exchange #1: R c Q_p n0_s."""
    c = len(shape)
    sb, qb = slab_bounds(shape[0], P), pencil_bounds(shape, P)
    return np.array([[R * c * (qb[p][1] - qb[p][0]) * (sb[s][1] - sb[s][0]) for p in range(P)] for s in range(P)])


def dist_env():
    import os

    return int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))


def broadcast_unique_id(make_id, group=None) -> bytes:
    """Rank 0 creates the NCCL unique id (make_id()), every rank receives it."""
    import torch.distributed as dist

    obj = [make_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def distributed_context(spec, device=None, group=None):
    """Context holding this rank's slab; the communicator spans the process group."""
    import torch.distributed as dist

    from . import _native

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    if device is None:
        device = dist_env()[2]
    uid = broadcast_unique_id(_native.nccl_unique_id, group)
    return _native.Context.distributed(spec, world, rank, device, uid)


def gather_slabs(local_full: np.ndarray, n0_axis: int, P: int, rank: int, group=None):
    """Each rank holds a full-layout array with only its planes valid (axis
    `n0_axis` is grid axis 0).  Returns the assembled array on rank 0, None elsewhere."""
    import torch
    import torch.distributed as dist

    bounds = slab_bounds(local_full.shape[n0_axis], P)
    lo, hi = bounds[rank]
    mine = torch.from_numpy(np.ascontiguousarray(np.take(local_full, range(lo, hi), axis=n0_axis)))
    parts = [None] * P if rank == 0 else None
    dist.gather_object(mine, parts, dst=0, group=group)
    if rank != 0:
        return None
    return np.concatenate([p.numpy() for p in parts], axis=n0_axis)

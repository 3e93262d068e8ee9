"""Multi-GPU application of the fast operator (one process per GPU).

Targets are sharded by contiguous Morton ranges cut at level-(L-1) block
boundaries (imq_ext_shard_bounds); every rank holds the full sorted point set
(setup is sub-second) and the full source vector.  After
imq_ext_operator_restrict a rank

  * forms the fine-level (L-1, L) moments of its own blocks and of the halo its
    far field reads (children of the 3x3 neighbourhoods of its blocks'
    parents) locally -- no exchange of fine moments or halo points;
  * forms the coarse-level (1..L-2) moments of its OWN points only; one
    all-reduce (sum) over NVLink of that coarse region (28 MB at config 4)
    makes them global;
  * evaluates the far + near field of its own targets.

gather_b() assembles the full product when a caller wants it.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from .capi import check, lib


def shard_bounds(leaf_start, levels: int, world: int, order: int | None = None) -> np.ndarray:
    """world+1 sorted-position bounds aligned to level-(L-1) blocks, balanced by
    point count, or by evaluation work when the expansion order is given."""
    ls = np.ascontiguousarray(leaf_start, dtype=np.int32)
    if ls.size != (1 << (2 * (levels + 1))) + 1:
        raise ValueError("leaf_start has the wrong length for `levels`")
    out = np.empty(world + 1, dtype=np.int32)
    lp, op = ls.ctypes.data_as(C.POINTER(C.c_int)), out.ctypes.data_as(C.POINTER(C.c_int))
    if order is None:
        check(lib().imq_ext_shard_bounds(lp, levels, world, op))
    else:
        check(lib().imq_ext_shard_bounds_work(lp, levels, order, world, op))
    return out


def leaf_start_from_keys(leaf_keys_sorted, levels: int) -> np.ndarray:
    """leaf_start (lower bounds) of a sorted array of finest Morton keys."""
    n_leaves = 1 << (2 * (levels + 1))
    return np.searchsorted(np.asarray(leaf_keys_sorted), np.arange(n_leaves + 1),
                           side="left").astype(np.int32)


class _DeviceView:
    """__cuda_array_interface__ view of library-owned device memory (float64)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                         "version": 3, "strides": None}


class ShardedOperator:
    """FastOperator whose moments and far/near evaluation cover this rank."""

    def __init__(self, op, rank: int, world: int):
        import torch
        self.op = op
        self.rank, self.world = rank, world
        self.bounds = shard_bounds(op.leaf_start(), op.levels, world, op.order)
        self.lo, self.hi = int(self.bounds[rank]), int(self.bounds[rank + 1])
        check(lib().imq_ext_operator_restrict(op.handle, self.lo, self.hi))
        self.perm = op.permutation()
        self.n_far, self.n_near = len(op.items("far")), len(op.items("near"))
        self.d_us = torch.empty(op.size, dtype=torch.float64, device="cuda")
        ptr, n = op.coarse_moments()
        self.coarse = torch.as_tensor(_DeviceView(ptr, n), device="cuda") if n else None

    def moments(self, d_u, stream=None, group=None, reduce=True):
        """Gather u, local + coarse-partial moments, coarse all-reduce, transform."""
        import torch.distributed as dist
        self.op.gather(d_u, self.d_us, stream)
        self.op.near_begin(self.d_us, stream)  # near field overlaps the moments + all-reduce
        self.op.moments_local(self.d_us, stream)
        if reduce and self.coarse is not None and self.world > 1:
            dist.all_reduce(self.coarse, group=group)
        if reduce:
            self.op.moments_finish(stream)

    def evaluate(self, d_b, stream=None):
        """b[perm[p]] for p in [lo, hi) (original order); other entries untouched."""
        self.op.far_near(self.d_us, d_b, (0, self.n_far), (0, self.n_near), stream, scatter=True)

    def apply_device(self, d_u, d_b, stream=None, group=None):
        self.moments(d_u, stream, group)
        self.evaluate(d_b, stream)

    def owned_original_indices(self) -> np.ndarray:
        return self.perm[self.lo:self.hi]


def gather_b(local_b, owned_idx, n: int, group=None):
    """Assemble the full product from every rank's owned entries (torch.distributed)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = local_b.device
    vals = local_b[torch.as_tensor(owned_idx, device=dev, dtype=torch.long)]
    sizes = [torch.zeros(1, dtype=torch.long, device=dev) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([vals.numel()], device=dev), group=group)
    m = int(max(s.item() for s in sizes))
    pad_v = torch.zeros(m, dtype=vals.dtype, device=dev)
    pad_i = torch.full((m,), -1, dtype=torch.long, device=dev)
    pad_v[:vals.numel()] = vals
    pad_i[:vals.numel()] = torch.as_tensor(owned_idx, device=dev, dtype=torch.long)
    all_v = [torch.empty_like(pad_v) for _ in range(world)]
    all_i = [torch.empty_like(pad_i) for _ in range(world)]
    dist.all_gather(all_v, pad_v, group=group)
    dist.all_gather(all_i, pad_i, group=group)
    out = torch.empty(n, dtype=vals.dtype, device=dev)
    for v, i in zip(all_v, all_i):
        k = i >= 0
        out[i[k]] = v[k]
    return out

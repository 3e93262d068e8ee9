"""Multi-GPU application of the fast operator (one process per GPU).

Targets are sharded by contiguous Morton ranges cut at level-(L-1) block
boundaries (imq_ext_shard_bounds); every rank holds the full sorted point set
(setup is sub-second).  After imq_ext_operator_restrict a rank

  * holds its own segment [lo, hi) of every Morton-ordered vector; one
    all-to-all per product (halo exchange, HaloExchange) brings in the source
    values of its halo leaves (imq_ext_operator_local_leaves: the leaves its
    fine moments and near field read) from the ranks that own them -- ~1 MB
    per rank at config 4 on 8 GPUs instead of the whole 134 MB vector;
  * forms the fine-level (L-1, L) moments of its own blocks and of the halo
    locally, and the coarse-level (1..L-2) moments of its OWN points only; one
    all-reduce (sum) over NVLink of that coarse region (28 MB at config 4)
    makes them global;
  * evaluates the far + near field of its own targets (apply_segment).

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


def leaf_positions(leaf_start, leaves) -> np.ndarray:
    """Sorted positions of the points of the given leaves (ascending leaves)."""
    ls = np.asarray(leaf_start, dtype=np.int64)
    lv = np.asarray(leaves, dtype=np.int64)
    if lv.size == 0:
        return np.empty(0, dtype=np.int64)
    a, b = ls[lv], ls[lv + 1]
    cnt = b - a
    starts = np.repeat(a - np.concatenate([[0], np.cumsum(cnt)[:-1]]), cnt)
    return starts + np.arange(int(cnt.sum()), dtype=np.int64)


def halo_plan(leaf_start, bounds, rank: int, local_leaves_by_rank):
    """Halo exchange plan of `rank` (pure host logic).

    local_leaves_by_rank[r]: the leaves rank r reads (own + halo).  Returns
    (send_idx, send_counts, recv_pos, recv_counts): send_idx are positions
    relative to this rank's segment start, grouped by destination rank;
    recv_pos are absolute sorted positions, grouped by source rank."""
    b = np.asarray(bounds, dtype=np.int64)
    lo, hi = int(b[rank]), int(b[rank + 1])
    world = len(b) - 1
    mine = leaf_positions(leaf_start, local_leaves_by_rank[rank])
    need = mine[(mine < lo) | (mine >= hi)]
    owner = np.searchsorted(b, need, side="right") - 1
    recv_pos = np.concatenate([need[owner == s] for s in range(world)]) if need.size else need
    recv_counts = [int(np.sum(owner == s)) for s in range(world)]
    send, send_counts = [], []
    for s in range(world):
        if s == rank:
            send_counts.append(0)
            continue
        theirs = leaf_positions(leaf_start, local_leaves_by_rank[s])
        mine_for_s = theirs[(theirs >= lo) & (theirs < hi)]
        send.append(mine_for_s - lo)
        send_counts.append(int(mine_for_s.size))
    send_idx = np.concatenate(send) if send else np.empty(0, dtype=np.int64)
    return send_idx.astype(np.int64), send_counts, recv_pos.astype(np.int64), recv_counts


class HaloExchange:
    """One all-to-all per product: every rank sends the values of its segment
    that other ranks' halos need (torch.distributed; NCCL on GPUs, gloo
    through host copies)."""

    def __init__(self, leaf_start, bounds, rank, local_leaves_by_rank, device, group=None):
        import torch
        import torch.distributed as dist
        si, sc, rp, rc = halo_plan(leaf_start, bounds, rank, local_leaves_by_rank)
        self.group = group
        self.host = dist.get_backend(group) == "gloo"
        self.send_idx = torch.as_tensor(si, device=device)
        self.recv_pos = torch.as_tensor(rp, device=device)
        self.send_counts, self.recv_counts = sc, rc
        self.bytes_sent = 8 * int(si.size)
        self.bytes_received = 8 * int(rp.size)

    def exchange(self, seg, full):
        """seg: this rank's segment; full: the Morton-ordered vector whose halo
        positions are filled (its own segment is written by the caller)."""
        import torch
        import torch.distributed as dist
        send = seg[self.send_idx]
        recv = torch.empty(int(sum(self.recv_counts)), dtype=seg.dtype, device=seg.device)
        if self.host:
            rh = recv.cpu()
            dist.all_to_all_single(rh, send.cpu(), self.recv_counts, self.send_counts,
                                   group=self.group)
            recv.copy_(rh)
        else:
            dist.all_to_all_single(recv, send, self.recv_counts, self.send_counts,
                                   group=self.group)
        full[self.recv_pos] = recv


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
        self.d_bs = torch.empty(op.size, dtype=torch.float64, device="cuda")
        self.halo = None

    def local_leaves(self) -> np.ndarray:
        """Leaves whose source values this rank reads (own + halo)."""
        lib_ = lib()
        n = C.c_size_t()
        check(lib_.imq_ext_operator_local_leaves(self.op.handle, None, 0, C.byref(n)))
        out = np.empty(n.value, dtype=np.int32)
        check(lib_.imq_ext_operator_local_leaves(self.op.handle,
                                                 out.ctypes.data_as(C.POINTER(C.c_int)),
                                                 n.value, C.byref(n)))
        return out

    def enable_halo(self, group=None):
        """Collective: builds the halo exchange plan (all ranks)."""
        import torch.distributed as dist
        mine = self.local_leaves()
        allv = [None] * self.world
        dist.all_gather_object(allv, mine, group=group)
        self.halo = HaloExchange(self.op.leaf_start(), self.bounds, self.rank, allv, "cuda", group)
        return self.halo

    def apply_segment(self, d_useg, d_bseg, stream=None, group=None):
        """Morton-ordered segment in, segment out: b_s[lo:hi] = (A u)_s[lo:hi]
        from u_s[lo:hi] (each rank its own), one halo all-to-all and one
        coarse-moment all-reduce per product."""
        import torch.distributed as dist
        if self.halo is None:
            raise RuntimeError("apply_segment: call enable_halo() first (collective)")
        self.d_us[self.lo:self.hi].copy_(d_useg)
        self.halo.exchange(d_useg, self.d_us)
        self.op.near_begin(self.d_us, stream)  # near field overlaps the moments + all-reduce
        self.op.moments_local(self.d_us, stream)
        if self.coarse is not None and self.world > 1:
            dist.all_reduce(self.coarse, group=group)
        self.op.moments_finish(stream)
        self.op.far_near(self.d_us, self.d_bs, (0, self.n_far), (0, self.n_near), stream)
        d_bseg.copy_(self.d_bs[self.lo:self.hi])

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

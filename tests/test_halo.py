"""Halo exchange of the sharded product (parallel.HaloExchange):
each rank holds only its Morton segment of the source vector and receives, in
one all-to-all, the values of the halo leaves its moments and near field read.

CPU (gloo, world 2): the plan from a host restatement of the restrict rule
(operator.cu setup_sharded_moments) fills exactly every position of each
rank's local leaves, and moves far fewer bytes than an all-gather.
GPU (gloo, two processes on one GPU, the NCCL path's code): apply_segment on
two ranks equals the unsharded product to 1e-13."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(fn, world, *args):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=fn, args=(r, world, port, q) + args) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return sorted(out, key=lambda x: x[0])


def local_leaves_rule(ls, L, lo, hi):
    """Host restatement of operator.cu setup_sharded_moments: non-empty
    children of the level-(L-1) blocks inside the 6x6 windows (grandparent
    neighbourhoods) of the rank's own level-(L-1) blocks."""
    def morton(i, j):
        k = 0
        for b in range(16):
            k |= ((i >> b) & 1) << (2 * b + 1) | ((j >> b) & 1) << (2 * b)
        return k

    def demorton(k):
        i = j = 0
        for b in range(16):
            i |= ((k >> (2 * b + 1)) & 1) << b
            j |= ((k >> (2 * b)) & 1) << b
        return i, j
    G = 1 << L
    own = [p for p in range(G * G) if ls[4 * p] >= lo and ls[4 * p + 4] <= hi and ls[4 * p] < hi]
    need = set()
    for p in own:
        pi, pj = demorton(p)
        gi, gj = pi >> 1, pj >> 1
        for a in range(max(0, 2 * gi - 2), min(G - 1, 2 * gi + 3) + 1):
            for b in range(max(0, 2 * gj - 2), min(G - 1, 2 * gj + 3) + 1):
                need.add(morton(a, b))
    leaves = []
    for p in sorted(need):
        for c in range(4):
            q = 4 * p + c
            if ls[q] < ls[q + 1]:
                leaves.append(q)
    return np.array(sorted(leaves), dtype=np.int64)


def _cpu_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2205_04194_b200.parallel import HaloExchange, leaf_positions
        rng = np.random.default_rng(3)
        L = 4
        n_leaves = 1 << (2 * (L + 1))
        counts = rng.poisson(20, n_leaves)
        counts[rng.random(n_leaves) < 0.1] = 0          # empty leaves
        ls = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        N = int(ls[-1])
        G = 1 << L
        cut = int(ls[4 * (G * G // 2)])                  # a level-(L-1) block boundary
        bounds = [0, cut, N]
        lists = [local_leaves_rule(ls, L, bounds[r], bounds[r + 1]) for r in range(world)]
        hx = HaloExchange(ls, bounds, rank, lists, "cpu")
        lo, hi = bounds[rank], bounds[rank + 1]
        seg = torch.arange(lo, hi, dtype=torch.float64)  # value = sorted position
        full = torch.full((N,), -1.0, dtype=torch.float64)
        full[lo:hi] = seg
        hx.exchange(seg, full)
        pos = leaf_positions(ls, lists[rank])
        ok = bool(torch.equal(full[torch.as_tensor(pos)], torch.as_tensor(pos, dtype=torch.float64)))
        q.put((rank, ok, hx.bytes_received, 8 * N))
    finally:
        dist.destroy_process_group()


def test_halo_plan_fills_local_leaves_cpu():
    res = _run(_cpu_worker, 2)
    for rank, ok, got, full in res:
        assert ok, rank
        assert 0 < got < full // 4  # a halo, not the vector


def _gpu_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2205_04194_b200 as P
        from paper_2205_04194_b200 import inputs
        from paper_2205_04194_b200.parallel import ShardedOperator
        torch.cuda.set_device(0)
        n = 1 << 18
        xy = inputs.uniform_points(n, 3)
        u = inputs.random_vector(n, 7)
        op = P.FastOperator(xy, 0.05, 12, 5)
        perm = torch.as_tensor(op.permutation().astype(np.int64), device="cuda")
        us = torch.as_tensor(u, device="cuda")[perm]
        sh = ShardedOperator(op, rank, world)
        hx = sh.enable_halo()
        seg = us[sh.lo:sh.hi].contiguous()
        out = torch.empty_like(seg)
        sh.apply_segment(seg, out)
        torch.cuda.synchronize()
        q.put((rank, sh.lo, sh.hi, out.cpu().numpy(), hx.bytes_received))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_apply_segment_two_ranks_matches_unsharded(imq):
    from paper_2205_04194_b200 import inputs
    n = 1 << 18
    xy = inputs.uniform_points(n, 3)
    u = inputs.random_vector(n, 7)
    with imq.FastOperator(xy, 0.05, 12, 5) as op:
        perm = op.permutation()
        b = op.apply(u)
    bs = b[perm]
    res = _run(_gpu_worker, 2)
    got = np.empty(n)
    for rank, lo, hi, seg, nbytes in res:
        got[lo:hi] = seg
        assert 0 < nbytes < 8 * n // 4
    assert float(np.max(np.abs(got - bs)) / np.max(np.abs(bs))) <= 1e-13

"""Multi-rank (world_size 2, gloo, CPU) coverage of the sharded application:
the product's shard_bounds / gather_b run on every rank, each rank evaluates
its own targets (with the oracle standing in for the GPU kernels, as the
checker), and the gathered product must equal the single-process one."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def morton(i, j):
    i = np.asarray(i, dtype=np.uint64)
    j = np.asarray(j, dtype=np.uint64)
    out = np.zeros_like(i)
    for b in range(16):
        out |= ((i >> np.uint64(b)) & np.uint64(1)) << np.uint64(2 * b + 1)
        out |= ((j >> np.uint64(b)) & np.uint64(1)) << np.uint64(2 * b)
    return out


def sorted_tree(oracle, xy, L):
    g = 1 << (L + 1)
    ids = oracle.block_ids(xy, L).astype(np.int64)
    keys = morton(ids // g, ids % g).astype(np.int64)
    perm = np.argsort(keys, kind="stable")
    from paper_2205_04194_b200.parallel import leaf_start_from_keys
    return perm, leaf_start_from_keys(keys[perm], L)


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import Oracle
        from paper_2205_04194_b200 import inputs
        from paper_2205_04194_b200.parallel import gather_b, shard_bounds
        O = Oracle()
        n, t, m, L = 4096, 0.1, 10, 2
        xy = inputs.uniform_points(n, 0)
        u = inputs.random_vector(n, 42)
        perm, ls = sorted_tree(O, xy, L)
        b = shard_bounds(ls, L, world)
        owned = perm[b[rank]:b[rank + 1]]
        local = torch.zeros(n, dtype=torch.float64)
        local[torch.as_tensor(owned)] = torch.as_tensor(O.fast_matvec_rows(xy, t, m, L, u, owned))
        full = gather_b(local, owned, n)
        ref = O.fast_matvec(xy, t, m, L, u)
        q.put((rank, bool(np.array_equal(full.numpy(), ref)), b.tolist()))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_sharded_product_matches_single(imq):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    b = res[0][2]
    assert b[0] == 0 and b[-1] == 4096 and b[0] < b[1] < b[2]


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_bounds_aligned_and_balanced(imq, oracle, world):
    from paper_2205_04194_b200 import inputs
    from paper_2205_04194_b200.parallel import shard_bounds
    for xy, L in ((inputs.uniform_points(20000, 0), 4), (inputs.gaussian_mixture(20000, 1), 4)):
        _, ls = sorted_tree(oracle, xy, L)
        b = shard_bounds(ls, L, world)
        parents = set(ls[::4].tolist())
        assert b[0] == 0 and b[-1] == 20000
        assert all(x in parents for x in b.tolist())          # cut at level-(L-1) blocks
        assert np.all(np.diff(b) >= 0)
        biggest = int(np.max(np.diff(ls[::4])))
        assert np.max(np.abs(np.diff(b) - 20000 / world)) <= biggest   # balanced to a block


def _morton(i, j):
    out = 0
    for b in range(16):
        out |= ((i >> b) & 1) << (2 * b + 1)
        out |= ((j >> b) & 1) << (2 * b)
    return out


def _parent_work(ls, L, M):
    """Independent restatement of the sharding work model: per level-(L-1)
    block, far (target, non-empty list block) pairs x (M^2+4M+12) + near
    pairs x 6 (interaction lists as partition.cpp:56-83); coarse levels
    weighted by the Chebyshev node share."""
    def count(l, i, j):
        q, sh = _morton(i, j), 2 * (L - l)
        return int(ls[(q + 1) << sh] - ls[q << sh])

    def nlist(l, i, j):
        g = 1 << (l + 1)
        if l == 1:
            cand = [(a, b) for a in range(g) for b in range(g)]
        else:
            pi, pj = i // 2, j // 2
            cand = [(a, b) for a in range(max(0, 2 * pi - 2), min(g, 2 * pi + 4))
                    for b in range(max(0, 2 * pj - 2), min(g, 2 * pj + 4))]
        return sum(1 for a, b in cand if max(abs(a - i), abs(b - j)) >= 2 and count(l, a, b) > 0)

    gL = 1 << (L + 1)
    w = np.zeros(1 << (2 * L))
    for p in range(1 << (2 * L)):
        far = near = 0
        for c in range(4):
            q = 4 * p + c
            nc = int(ls[q + 1] - ls[q])
            if not nc:
                continue
            i = j = 0
            for b in range(16):
                i |= ((q >> (2 * b + 1)) & 1) << b
                j |= ((q >> (2 * b)) & 1) << b
            f = nlist(L, i, j)
            for l in range(1, L):  # levels 1..L-2 through 20x20 Chebyshev nodes when L >= 4
                il, jl = i >> (L - l), j >> (L - l)
                wl = min(1.0, 400.0 / count(l, il, jl)) if (L >= 4 and l <= L - 2) else 1.0
                f += wl * nlist(l, il, jl)
            f += 1.4 if L >= 4 else 0.0
            far += nc * f
            near += nc * sum(count(L, a, b) for a in range(max(0, i - 1), min(gL, i + 2))
                             for b in range(max(0, j - 1), min(gL, j + 2)))
        w[p] = (M * M + 4 * M + 12) * far + 6 * near
    return w


@pytest.mark.parametrize("world", [2, 3, 8])
def test_shard_bounds_balanced_by_work(imq, oracle, world):
    from paper_2205_04194_b200 import inputs
    from paper_2205_04194_b200.parallel import shard_bounds
    L, M = 4, 12
    for xy in (inputs.uniform_points(20000, 0), inputs.gaussian_mixture(20000, 1)):
        _, ls = sorted_tree(oracle, xy, L)
        b = shard_bounds(ls, L, world, order=M)
        parents = ls[::4]
        assert b[0] == 0 and b[-1] == 20000 and np.all(np.diff(b) >= 0)
        assert all(x in set(parents.tolist()) for x in b.tolist())
        w = _parent_work(ls, L, M)
        cum = np.concatenate([[0.0], np.cumsum(w)])
        at = np.searchsorted(parents, b, side="left")     # parent index of each cut
        share = np.diff(cum[at])
        assert np.max(np.abs(share - cum[-1] / world)) <= np.max(w) + 1e-6

"""Multi-process (gloo, world_size 2, CPU) tests of the multi-GPU layer's host logic as the library
implements it: every rank asks libmch.so for its sharding plan (`mch_shard_plan`, host only: no
GPU), and the ranks then run exchange step (i) of SURVEY.md §8(e) over gloo exactly as the library
does over NCCL — after each level every transfer (macropoint, src, dst) of the plan moves that
parent's "solution" from src to dst — and check that every child finds all its parents
(Eq. 11) locally, that the owned sets partition every S_n, that the ranks agree on the plan, and
that the owner-masked sum of exchange step (ii) is exact."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

CASES = [  # d, n, N, M, L, eta
    (2, 64, 2, 8, 3, 2),
    (3, 32, 2, 4, 2, 2),
    (2, 1024, 2, 32, 3, 2),   # BASELINE config 2 geometry
    (3, 256, 2, 16, 4, 2),    # BASELINE config 5 geometry
]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _hierarchy(d, n, M, L, eta):
    """every child's parents, each macropoint's level and S_n, from the oracle's planner (an
    independent implementation; pinned in tests/test_oracle_planner.py)"""
    from oracle.planner import Plan
    pl = Plan(d, n, M, L, eta)
    par = {}
    for lev in range(2, L + 1):
        for k in pl.S(lev):
            par[pl.linear_index(k)] = [pl.linear_index(t) for t, _ in pl.parents(k)]
    lev_of = {pl.linear_index(k): lev for lev in range(1, L + 1) for k in pl.S(lev)}
    S = {lev: sorted(pl.linear_index(k) for k in pl.S(lev)) for lev in range(1, L + 1)}
    return par, lev_of, S


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2503_01276_b200.api import mch_shard_plan
    out = []
    for (d, n, N, M, L, eta) in CASES:
        par, lev_of, S = _hierarchy(d, n, M, L, eta)
        owned, xfers = {}, {}
        for lev in range(1, L + 1):
            o, x = mch_shard_plan(d, n, N, M, L, eta, rank, world, lev)
            owned[lev], xfers[lev] = o.tolist(), x
        ok = True
        # (a) the owned sets partition S_n (all-gather of the owned lists)
        for lev in range(1, L + 1):
            allo = [None] * world
            dist.all_gather_object(allo, owned[lev])
            flat = sorted(m for o in allo for m in o)
            ok &= flat == S[lev]
            # contiguous runs in lexicographic order, rank r before rank r+1
            pos = {m: i for i, m in enumerate(S[lev])}
            for r in range(world):
                ps = [pos[m] for m in allo[r]]
                ok &= ps == list(range(ps[0], ps[0] + len(ps))) if ps else True
            # (b) every rank lists the same transfers
            allx = [None] * world
            dist.all_gather_object(allx, xfers[lev].tolist())
            ok &= all(a == allx[0] for a in allx)
        # (c) exchange step (i) over gloo, "solutions" = 3 recognisable values per macropoint
        have = {}
        for lev in range(1, L + 1):
            for m in owned[lev]:
                have[m] = torch.tensor([m, m + 0.5, -m], dtype=torch.float64)
            reqs = []
            for m, src, dst in xfers[lev].tolist():
                if src == rank:
                    reqs.append(dist.isend(have[m], dst))
                elif dst == rank:
                    buf = torch.empty(3, dtype=torch.float64)
                    reqs.append(dist.irecv(buf, src))
                    have[m] = buf
            for r in reqs:
                r.wait()
        for lev in range(2, L + 1):
            for m in owned[lev]:
                for t in par[m]:
                    ok &= t in have and torch.equal(have[t], torch.tensor([t, t + 0.5, -t], dtype=torch.float64))
        # nothing is received that no owned child needs
        need = {t for lev in range(2, L + 1) for m in owned[lev] for t in par[m]}
        recv = {m for lev in range(1, L + 1) for m, s_, d_ in xfers[lev].tolist() if d_ == rank}
        ok &= recv <= need
        # (d) exchange step (ii): owner-masked sum is exact
        P = sum(len(v) for v in S.values())
        G = torch.zeros((P, 2, 2), dtype=torch.float64)
        for lev in range(1, L + 1):
            for m in owned[lev]:
                G[m] = torch.tensor([[m + 0.1, 1.0 / (m + 3)], [1.0 / (m + 3), m * 1e-17 + 1.0]], dtype=torch.float64)
        dist.all_reduce(G)
        for m in range(P):
            ok &= torch.equal(G[m], torch.tensor([[m + 0.1, 1.0 / (m + 3)], [1.0 / (m + 3), m * 1e-17 + 1.0]],
                                                 dtype=torch.float64))
        out.append(bool(ok))
    q.put((rank, out))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_library_shard_plan_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(all(r[1]) for r in res), res


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_plan_balance(world):
    """cost-balanced ownership: config 5 at 8 ranks, every rank's share of each level's work
    (window nodes) within one macropoint's work of the mean"""
    from paper_2503_01276_b200.api import mch_shard_plan
    from oracle.planner import Plan
    d, n, N, M, L, eta = 3, 256, 2, 16, 4, 2
    pl = Plan(d, n, M, L, eta)
    for lev in range(1, L + 1):
        s = eta ** (lev - 1)

        def work(k):
            lo, hi = pl.window(k)
            return int(np.prod([(hi[i] - lo[i]) // s + 1 for i in range(d)]))
        wl = {pl.linear_index(k): work(k) for k in pl.S(lev)}
        shares = []
        for r in range(world):
            o, _ = mch_shard_plan(d, n, N, M, L, eta, r, world, lev)
            shares.append(sum(wl[m] for m in o.tolist()))
        assert sum(shares) == sum(wl.values())
        assert max(shares) - sum(shares) / world <= max(wl.values()), (lev, shares)

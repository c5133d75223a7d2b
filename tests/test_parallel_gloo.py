"""Multi-process (gloo, world_size 2, CPU) tests of the multi-GPU layer's exchange logic
(paper_2503_01276_b200/parallel.py): owner chunks of the parent pool, their broadcast, and the
exact owner-masked all-reduce of the coefficient tensors.  The CUDA library is not needed:
the functions operate on torch tensors and a pool layout replicated here from mch.h's
contract (by level, then owner = position mod world, then lexicographic)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

def _import_parallel():
    # parallel.py imports only torch; import it without loading libmch.so
    import importlib.util
    import sys
    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("mch_parallel", os.path.join(here, "paper_2503_01276_b200", "parallel.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules["mch_parallel"] = mod
    spec.loader.exec_module(mod)
    return mod


def _layout(levels_pts, sizes, world, L):
    """pool offsets as libmch lays them out (mch_create)"""
    off, slots = 0, {}
    for lev in range(1, L):
        pts = levels_pts[lev]
        for owner in range(world):
            for m in pts[owner::world]:
                slots[m] = (off, sizes[m])
                off += sizes[m]
    return slots, off


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    par = _import_parallel()
    L = 3
    levels = {1: [0, 4, 8], 2: [2, 6, 10, 12, 14], 3: [1, 3, 5, 7, 9, 11, 13]}
    sizes = {m: 3 + (m % 4) for m in range(15)}
    slots, n = _layout(levels, sizes, world, L)
    pool = torch.zeros(n, dtype=torch.float64)
    # each rank "solves" its own macropoints of level 1 and 2: fill with recognisable values
    for lev in (1, 2):
        for m in levels[lev][rank::world]:
            o, ln = slots[m]
            pool[o:o + ln] = torch.arange(ln, dtype=torch.float64) + 100.0 * m
    for lev in (1, 2):
        chunks = par.owner_chunks(levels[lev], lambda m: slots.get(m, (-1, 0)), world)
        par.exchange_chunks(pool, chunks)
    ok = True
    for lev in (1, 2):
        for m in levels[lev]:
            o, ln = slots[m]
            ok &= torch.equal(pool[o:o + ln], torch.arange(ln, dtype=torch.float64) + 100.0 * m)
    okp = bool(ok)
    # coefficients: owned entries only, exact all-reduce
    P, nr = 15, 2
    G = torch.full((P, nr, nr), float("nan"), dtype=torch.float64)  # garbage where not owned
    owned = torch.zeros(P, dtype=torch.bool)
    for lev in (1, 2, 3):
        for m in levels[lev][rank::world]:
            owned[m] = True
            G[m] = torch.tensor([[m + 0.1, 1.0 / (m + 3)], [1.0 / (m + 3), m * 1e-17 + 1.0]], dtype=torch.float64)
    out = par.gather_coeffs(G, owned)
    for m in range(P):
        ok &= torch.equal(out[m], torch.tensor([[m + 0.1, 1.0 / (m + 3)], [1.0 / (m + 3), m * 1e-17 + 1.0]],
                                                dtype=torch.float64))
    q.put((rank, bool(ok), okp))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_exchange_and_gather_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] for r in res), res


def test_owner_chunks_contiguity():
    par = _import_parallel()
    levels = {1: [0, 4, 8, 12], 2: [2, 6, 10]}
    sizes = {m: 5 + m for m in range(13)}
    for world in (1, 2, 3, 4):
        slots, n = _layout({1: levels[1], 2: levels[2]}, sizes, world, 3)
        for lev in (1, 2):
            ch = par.owner_chunks(levels[lev], lambda m: slots.get(m, (-1, 0)), world)
            covered = sum(hi - lo for _, lo, hi in ch)
            assert covered == sum(sizes[m] for m in levels[lev])
            assert len({o for o, _, _ in ch}) == len(ch)

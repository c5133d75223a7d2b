"""The library's multi-GPU sharding on ONE GPU (no NCCL): contexts of rank 0..world-1 solve their
shards (params.rank/world); between levels the test moves exactly the pool slots the library's
plan lists (mch_shard_plan, the same transfers the NCCL path sends) from the owner's context to the
receiver's; the owner-masked coefficient tensors are summed.  The result must equal the world = 1
run BITWISE (per-macropoint work is rank-independent), and a transfer left out
must show up (the pool of a world > 1 context is poisoned with NaN).  Also checks the library's
own comm-less behaviour: non-owned coefficients are 0."""
import numpy as np
import pytest

from tests.test_gpu_parity import _admissible

pytestmark = pytest.mark.gpu


class _Dev:
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3,
                                         "strides": None}


def _view(ptr, n):
    import torch
    return torch.as_tensor(_Dev(ptr, n), device="cuda")


def _run(d, n, N, M, L, kap, ids, world, drop=None):
    import torch
    from paper_2503_01276_b200 import Homogenizer
    from paper_2503_01276_b200.api import mch_shard_plan
    hs = [Homogenizer(d, n, N, M, L, 2, kap, ids, rank=r, world=world) for r in range(world)]
    pools = []
    for h in hs:
        ptr, ln = h.pool_info()
        pools.append(_view(ptr, ln) if ln > 0 else None)
    moved = 0
    for lev in range(1, L + 1):
        for h in hs:
            h.solve_level(lev)
        if world > 1 and lev < L:
            _, xf = mch_shard_plan(d, n, N, M, L, 2, 0, world, lev)
            for m, src, dst in xf.tolist():
                if drop is not None and moved == drop:
                    moved += 1
                    continue
                o, ln = hs[src].pool_slot(m)
                o2, ln2 = hs[dst].pool_slot(m)
                assert ln == ln2 > 0
                pools[dst][o2:o2 + ln].copy_(pools[src][o:o + ln])
                moved += 1
            torch.cuda.synchronize()
    G = None
    for r, h in enumerate(hs):
        Gr = h.effective_coeffs()
        owned = np.zeros(h.num_macropoints, dtype=bool)
        for lev in range(1, L + 1):
            o, _ = mch_shard_plan(d, n, N, M, L, 2, r, world, lev)
            owned[o] = True
        assert np.all(Gr[~owned] == 0.0)  # no communicator: other ranks' entries stay 0
        G = Gr if G is None else G + Gr
    for h in hs:
        h.close()
    return G, moved


@pytest.mark.parametrize("d,n,M,L,N,world", [(2, 64, 8, 3, 2, 2), (2, 64, 8, 3, 2, 3), (3, 32, 4, 2, 2, 2),
                                              (3, 16, 4, 2, 2, 4)])
def test_sharded_equals_single_bitwise(d, n, M, L, N, world):
    kap, ids = _admissible(d, n, M, N, 77 + d)
    G1, _ = _run(d, n, N, M, L, kap, ids, 1)
    Gw, moved = _run(d, n, N, M, L, kap, ids, world)
    assert moved > 0
    assert np.array_equal(G1, Gw)


def test_missing_transfer_is_detected():
    d, n, M, L, N = 2, 64, 8, 3, 2
    kap, ids = _admissible(d, n, M, N, 79)
    G1, _ = _run(d, n, N, M, L, kap, ids, 1)
    try:
        Gw, _ = _run(d, n, N, M, L, kap, ids, 2, drop=0)
    except RuntimeError:
        return  # NaN parent -> PCG breakdown reported (MCH_ENOCONV)
    assert not np.array_equal(G1, Gw) and not np.all(np.isfinite(Gw))


def test_library_nccl_single_rank():
    """The library's NCCL path on one GPU: mch_comm_id / mch_comm_init (NCCL resolved at run time from
    libnccl.so.2) build a one-rank communicator; a context created with it runs the collective
    mch_effective_coeffs (ncclAllReduce) and must return the same coefficients, bitwise, as a
    context without one.  (The point-to-point parent exchange needs >= 2 GPUs.)"""
    import torch
    from paper_2503_01276_b200 import Homogenizer
    from paper_2503_01276_b200.api import mch_comm_destroy, mch_comm_id, mch_comm_init
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    d, n, M, L, N = 2, 64, 8, 3, 2
    kap, ids = _admissible(d, n, M, N, 81)
    with Homogenizer(d, n, N, M, L, 2, kap, ids) as h:
        h.solve_all()
        G0 = h.effective_coeffs()
    uid = mch_comm_id()
    assert len(uid) == 128
    comm = mch_comm_init(1, 0, uid)
    try:
        with Homogenizer(d, n, N, M, L, 2, kap, ids, comm=comm) as h:
            h.solve_all()
            G1 = h.effective_coeffs()
    finally:
        mch_comm_destroy(comm)
    assert np.array_equal(G0, G1)

"""Multi-GPU layer: one process per GPU, macropoints of every level sharded across ranks.

The method has exactly two exchange steps:
  (i) after level n, the fine local solutions of the level-n parents (T_{L-1}) are needed by
      children of later levels on every rank — each owner broadcasts its contiguous pool
      chunk (the library lays the pool out by (level, owner)) over NCCL;
  (ii) at the end the Eq. (7) coefficient tensors are combined: non-owned entries are exactly
      zero, so an all-reduce(SUM) reproduces the single-GPU tensor bit for bit.
Everything else is independent per macropoint ("independent across different
macropoints").  torch.distributed (NCCL over NVLink/NVSwitch; gloo in the CPU tests) is the
plumbing; the compute stays in libmch.so.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


class _CudaArray:
    """__cuda_array_interface__ view of library-owned device memory (float64)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                         "version": 3, "strides": None}


def device_view(ptr: int, n: int) -> torch.Tensor:
    return torch.as_tensor(_CudaArray(ptr, n), device="cuda")


def owner_chunks(level_points, slots, world):
    """[(owner, lo, hi)] contiguous pool ranges produced by each owner at one level.
    level_points: lexicographic indices of S_n in solve order; slots: idx -> (offset, length)."""
    out = []
    for owner in range(world):
        spans = [slots(m) for m in level_points[owner::world]]
        spans = [(o, n) for o, n in spans if o >= 0 and n > 0]
        if not spans:
            continue
        lo = min(o for o, _ in spans)
        hi = max(o + n for o, n in spans)
        assert hi - lo == sum(n for _, n in spans), "pool chunk of an owner must be contiguous"
        out.append((owner, lo, hi))
    return out


def exchange_chunks(pool: torch.Tensor, chunks, group=None):
    """Broadcast every owner's chunk to all ranks (exchange step (i))."""
    for owner, lo, hi in chunks:
        dist.broadcast(pool[lo:hi], src=owner, group=group)


def gather_coeffs(G: torch.Tensor, owned: torch.Tensor, group=None):
    """Exchange step (ii): each rank contributes only its own macropoints (others exactly 0),
    so the all-reduce(SUM) is exact.  G: [P, n_rhs, n_rhs]; owned: bool [P]."""
    out = torch.where(owned[:, None, None], G, torch.zeros((), dtype=G.dtype, device=G.device))
    dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
    return out


class ShardedHomogenizer:
    """Homogenizer over `world` ranks (one GPU each); same results as one GPU, bitwise."""

    def __init__(self, cfg_or_args, kappa, ids, rank, world, group=None, **kw):
        from .api import Homogenizer
        if isinstance(cfg_or_args, tuple):
            self.h = Homogenizer(*cfg_or_args, kappa, ids, rank=rank, world=world, **kw)
        else:
            self.h = Homogenizer.from_config(cfg_or_args, kappa, ids, rank=rank, world=world, **kw)
        self.rank, self.world, self.group = rank, world, group
        ptr, n = self.h.pool_info()
        self.pool = device_view(ptr, n) if n > 0 else None
        self.G = device_view(self.h.coeffs_device_ptr(), self.h.num_macropoints * self.h.n_rhs ** 2)
        self.chunks = {}
        owned = torch.zeros(self.h.num_macropoints, dtype=torch.bool)
        for lev in range(1, self.h.L + 1):
            pts = self.h.level_macropoints(lev)
            owned[pts[rank::world]] = True
            if lev < self.h.L:
                self.chunks[lev] = owner_chunks(pts, self.h.pool_slot, world)
        self.owned = owned.to(self.G.device)

    def reset(self):
        self.h.reset()

    def set_medium(self, kappa, ids):
        self.h.set_medium(kappa, ids)

    def solve_all(self):
        for lev in range(1, self.h.L + 1):
            self.h.solve_level(lev)
            if self.world > 1 and lev < self.h.L:
                exchange_chunks(self.pool, self.chunks[lev], self.group)

    def effective_coeffs(self):
        G = self.G.view(self.h.num_macropoints, self.h.n_rhs, self.h.n_rhs)
        if self.world > 1:
            return gather_coeffs(G, self.owned, self.group)
        return G

    def close(self):
        self.h.close()

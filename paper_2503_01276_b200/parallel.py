"""Multi-GPU layer: one process per GPU, the macropoints of every level sharded across ranks.

The method has exactly two exchange steps:
  (i)  after level n, the fine local solutions of the level-n parents go to the ranks whose
       children of later levels read them (Eq. 11);
  (ii) at the end the Eq. (7) coefficient tensors are combined (non-owned entries are exactly 0,
       so an all-reduce reproduces the single-GPU tensor bit for bit).
Everything else is independent per macropoint.  Both steps run INSIDE libmch.so
on its NCCL communicator (grouped ncclSend/ncclRecv of whole pool slots per the library's
sharding plan, `mch_shard_plan`; ncclAllReduce of the coefficients), so mch_solve_level and
mch_effective_coeffs are collective.  torch.distributed is plumbing only: it broadcasts the NCCL
unique id once.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .api import Homogenizer, mch_comm_destroy, mch_comm_id, mch_comm_init


def library_comm(rank: int, world: int, group=None):
    """NCCL communicator of the library for this rank (id from rank 0 via torch.distributed)."""
    obj = [mch_comm_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return mch_comm_init(world, rank, obj[0])


class ShardedHomogenizer:
    """Homogenizer over `world` ranks (one GPU each); same results as one GPU, bitwise."""

    def __init__(self, cfg_or_args, kappa, ids, rank, world, group=None, **kw):
        self.rank, self.world, self.group = rank, world, group
        self.comm = library_comm(rank, world, group) if world > 1 else None
        if isinstance(cfg_or_args, tuple):
            self.h = Homogenizer(*cfg_or_args, kappa, ids, rank=rank, world=world, comm=self.comm, **kw)
        else:
            self.h = Homogenizer.from_config(cfg_or_args, kappa, ids, rank=rank, world=world, comm=self.comm, **kw)
        self._G = None

    def reset(self):
        self.h.reset()

    def set_medium(self, kappa, ids):
        self.h.set_medium(kappa, ids)

    def solve_all(self):
        self.h.solve_all()  # collective per level (exchange step (i) inside the library)

    def effective_coeffs(self, out=None):
        """[P, n_rhs, n_rhs] on every rank (exchange step (ii) inside the library); out may be a
        device tensor or (pinned) host memory."""
        if out is None:
            if self._G is None:
                self._G = torch.empty((self.h.num_macropoints, self.h.n_rhs, self.h.n_rhs), dtype=torch.float64,
                                      device="cuda")
            out = self._G
        return self.h.effective_coeffs(out)

    def close(self):
        self.h.close()
        if self.comm is not None:
            mch_comm_destroy(self.comm)
            self.comm = None

"""Thin Python API over the C ABI (include/mch.h).

Names follow the ABI: ``mch_create`` / ``mch_solve_level`` / ``mch_effective_coeffs`` wrap
the C calls one-to-one; :class:`Homogenizer` bundles them.  Inputs may be host numpy
arrays or CUDA torch tensors; PyTorch is only used for device memory and the stream.
"""
from __future__ import annotations

import ctypes
import json
import os

import numpy as np

from . import _native
from ._native import MchLevelStats, MchParams, check, lib


def _ptr(a):
    """(pointer, on_device) of a numpy array or torch tensor (must be contiguous)."""
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data, 0
    import torch
    if isinstance(a, torch.Tensor):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return a.data_ptr(), int(a.is_cuda)
    raise TypeError(type(a))


def _current_stream():
    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.current_stream().cuda_stream
    except Exception:  # pragma: no cover
        pass
    return None


INTERP = {"dlinear": 0, "nearest_s1": 1, "physical_s1": 2}
LAYOUT = {"vertex": 0, "block": 1}


def mch_create(d, n, num_continua, M, levels, eta, kappa, continuum_id, oversample=1, rtol=1e-12,
               max_iter=20000, rank=0, world=1, keep_all=False, stream=None, interp="dlinear",
               layout="vertex", allocator=None, comm=None):
    """Returns an opaque context handle (ctypes.c_void_p).  allocator: None (cudaMalloc) or an
    (alloc, free) pair of _native.ALLOC_FN / FREE_FN callbacks, e.g. _native.torch_allocator()."""
    if isinstance(kappa, np.ndarray):
        kappa = np.ascontiguousarray(kappa, dtype=np.float64)
        continuum_id = np.ascontiguousarray(continuum_id, dtype=np.uint8)
    kp, kdev = _ptr(kappa)
    ip, idev = _ptr(continuum_id)
    if kdev != idev:
        raise ValueError("kappa and continuum_id must both be host or both be device buffers")
    p = MchParams(d=d, n=n, num_continua=num_continua, M=M, levels=levels, eta=eta,
                  oversample=oversample, rtol=rtol, max_iter=max_iter, rank=rank, world=world,
                  keep_all=int(keep_all), stream=stream if stream is not None else _current_stream(),
                  interp=INTERP[interp], layout=LAYOUT[layout], nccl_comm=comm)
    if allocator is not None:
        p.alloc = ctypes.cast(allocator[0], ctypes.c_void_p)
        p.free = ctypes.cast(allocator[1], ctypes.c_void_p)
    ctx = ctypes.c_void_p()
    check(lib.mch_create(ctypes.byref(p), kp, ip, kdev, ctypes.byref(ctx)), None)
    return ctx


def mch_set_medium(ctx, kappa, continuum_id):
    """New medium into an existing context (plan and buffers reused); host or device inputs."""
    if isinstance(kappa, np.ndarray):
        kappa = np.ascontiguousarray(kappa, dtype=np.float64)
        continuum_id = np.ascontiguousarray(continuum_id, dtype=np.uint8)
    kp, kdev = _ptr(kappa)
    ip, idev = _ptr(continuum_id)
    if kdev != idev:
        raise ValueError("kappa and continuum_id must both be host or both be device buffers")
    check(lib.mch_set_medium(ctx, kp, ip, kdev), ctx)


def mch_solve_level(ctx, level):
    check(lib.mch_solve_level(ctx, level), ctx)


def mch_effective_coeffs(ctx, out):
    op, odev = _ptr(out)
    n = out.numel() if hasattr(out, "numel") else out.size
    check(lib.mch_effective_coeffs(ctx, op, n, odev), ctx)
    return out


def mch_set_source(ctx, f):
    """Source f (cellwise, n^d) for the Eq. (7) load vectors; None removes it."""
    if f is None:
        check(lib.mch_set_source(ctx, None, 0), ctx)
        return
    if isinstance(f, np.ndarray):
        f = np.ascontiguousarray(f, dtype=np.float64)
    fp, fdev = _ptr(f)
    check(lib.mch_set_source(ctx, fp, fdev), ctx)


def mch_load_vectors(ctx, out):
    op, odev = _ptr(out)
    n = out.numel() if hasattr(out, "numel") else out.size
    check(lib.mch_load_vectors(ctx, op, n, odev), ctx)
    return out


def mch_macro_solve(ctx, out, G=None, b=None, rtol=1e-12, max_iter=0):
    """Upscaled system (Eq. 6) into out [N][(M+1)^d]; G, b default to the context's own.
    Returns the PCG iteration count."""
    gp = bp = None
    gdev = 0
    if G is not None:
        if isinstance(G, np.ndarray):
            G = np.ascontiguousarray(G, dtype=np.float64)
            b = np.ascontiguousarray(b, dtype=np.float64)
        gp, gdev = _ptr(G)
        bp, bdev = _ptr(b)
        if gdev != bdev:
            raise ValueError("G and b must both be host or both be device buffers")
    op, odev = _ptr(out)
    n = out.numel() if hasattr(out, "numel") else out.size
    it = ctypes.c_int(0)
    check(lib.mch_macro_solve(ctx, gp, bp, gdev, op, n, odev, rtol, max_iter, ctypes.byref(it)), ctx)
    return it.value


def mch_destroy(ctx):
    lib.mch_destroy(ctx)


def mch_comm_id():
    """A new NCCL unique id (128 bytes) — on one rank; broadcast it to the others."""
    buf = ctypes.create_string_buffer(128)
    check(lib.mch_comm_id(buf, 128), None)
    return buf.raw


def mch_comm_init(world, rank, uid):
    """ncclComm_t of this rank (collective; call after torch.cuda.set_device)."""
    comm = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(bytes(uid), 128)
    check(lib.mch_comm_init(ctypes.byref(comm), world, rank, buf, 128), None)
    return comm.value


def mch_comm_destroy(comm):
    check(lib.mch_comm_destroy(comm), None)


def mch_shard_plan(d, n, N, M, L, eta, rank, world, level, l=1, interp="dlinear", layout="vertex"):
    """Host-only sharding plan (no GPU): (owned lexicographic indices of S_level on this rank,
    transfers [k, 3] = (macropoint, src, dst) sent after level `level`)."""
    p = MchParams(d=d, n=n, num_continua=N, M=M, levels=L, eta=eta, oversample=l, rtol=1e-12,
                  max_iter=0, rank=rank, world=world, keep_all=0, stream=None,
                  interp=INTERP[interp], layout=LAYOUT[layout])
    no, nx = ctypes.c_int64(0), ctypes.c_int64(0)
    check(lib.mch_shard_plan(ctypes.byref(p), level, None, 0, ctypes.byref(no), None, 0, ctypes.byref(nx)), None)
    owned = np.zeros(max(no.value, 1), dtype=np.int64)
    xf = np.zeros((max(nx.value, 1), 3), dtype=np.int64)
    check(lib.mch_shard_plan(ctypes.byref(p), level, owned.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                             owned.size, ctypes.byref(no), xf.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                             xf.shape[0], ctypes.byref(nx)), None)
    return owned[:no.value], xf[:nx.value]


class Homogenizer:
    """Hierarchical multicontinuum homogenization hot path on one GPU (or one rank's shard)."""

    def __init__(self, d, n, N, M, L, eta, kappa, ids, l=1, rtol=1e-12, max_iter=20000, rank=0,
                 world=1, keep_all=False, stream=None, interp="dlinear", layout="vertex",
                 torch_memory=False, comm=None):
        self.d, self.n, self.N, self.M, self.L, self.eta, self.l = d, n, N, M, L, eta, l
        self.interp = interp
        self.rank, self.world = rank, world
        self.n_rhs = N * (1 + d)
        self.mv = M + 1 if layout == "vertex" else M  # macropoints per dimension
        self.num_macropoints = self.mv ** d
        # torch_memory: every device buffer of the context comes from PyTorch's caching allocator
        self._allocator = _native.torch_allocator() if torch_memory else None
        self.ctx = mch_create(d, n, N, M, L, eta, kappa, ids, oversample=l, rtol=rtol,
                              max_iter=max_iter, rank=rank, world=world, keep_all=keep_all,
                              stream=stream, interp=interp, layout=layout, allocator=self._allocator,
                              comm=comm)
        self.solved = 0

    @classmethod
    def from_config(cls, cfg, kappa, ids, **kw):
        return cls(cfg.d, cfg.n, cfg.N, cfg.M, cfg.L, cfg.eta, kappa, ids, l=cfg.l, **kw)

    def solve_level(self, level):
        mch_solve_level(self.ctx, level)
        self.solved = level

    def reset(self):
        check(lib.mch_reset(self.ctx), self.ctx)
        self.solved = 0

    def set_medium(self, kappa, ids):
        mch_set_medium(self.ctx, kappa, ids)
        self.solved = 0

    def solve_all(self, log=None):
        """Solve the remaining levels in order.  `log`: path of a JSON-lines
        file that gets one record per level (mch_get_level_stats of that solve: macropoints,
        iterations, per-phase device times, bytes, launches), or the MCH_LEVEL_LOG environment
        variable; appended, one line per level."""
        log = log or os.environ.get("MCH_LEVEL_LOG")
        for lev in range(self.solved + 1, self.L + 1):
            self.solve_level(lev)
            if log:
                rec = {"level": lev, "d": self.d, "n_rhs": self.n_rhs, "rank": self.rank, "world": self.world}
                rec.update(self.level_stats(lev))
                with open(log, "a") as f:
                    f.write(json.dumps(rec) + "\n")

    def effective_coeffs(self, out=None):
        if out is None:
            out = np.zeros((self.num_macropoints, self.n_rhs, self.n_rhs))
        return mch_effective_coeffs(self.ctx, out)

    def set_source(self, f):
        """NEXT-2: source term for the load vectors (before solve_all)."""
        mch_set_source(self.ctx, f)

    def load_vectors(self, out=None):
        if out is None:
            out = np.zeros((self.num_macropoints, self.N))
        return mch_load_vectors(self.ctx, out)

    def macro_solve(self, G=None, b=None, out=None, rtol=1e-12, max_iter=0):
        """U [N][(M+1)^d] of the upscaled system (block layout).  Returns (U, iterations)."""
        if out is None:
            out = np.zeros((self.N, (self.M + 1) ** self.d))
        it = mch_macro_solve(self.ctx, out, G, b, rtol=rtol, max_iter=max_iter)
        return out, it

    def fine_solve(self, f, rtol=1e-10, max_iter=0, out=None):
        """NEXT-3: global fine reference solution of Eq. (2) with this context's kappa and the
        cellwise source f.  Returns (u nodal [(n+1)^d], iterations)."""
        if isinstance(f, np.ndarray):
            f = np.ascontiguousarray(f, dtype=np.float64)
        fp, fdev = _ptr(f)
        if out is None:
            out = np.zeros(((self.n + 1),) * self.d)
        op, odev = _ptr(out)
        n = out.numel() if hasattr(out, "numel") else out.size
        it = ctypes.c_int(0)
        check(lib.mch_fine_solve(self.ctx, fp, fdev, op, n, odev, rtol, max_iter, ctypes.byref(it)), self.ctx)
        return out, it.value

    def fine_block_averages(self, u, out=None):
        """[P][N]: (1/|K_p cap Omega_i|) int_{K_p cap Omega_i} u."""
        if isinstance(u, np.ndarray):
            u = np.ascontiguousarray(u, dtype=np.float64)
        up, udev = _ptr(u)
        if out is None:
            out = np.zeros((self.num_macropoints, self.N))
        op, odev = _ptr(out)
        n = out.numel() if hasattr(out, "numel") else out.size
        check(lib.mch_fine_block_averages(self.ctx, up, udev, op, n, odev), self.ctx)
        return out

    def save_checkpoint(self, path):
        """mch_checkpoint_save: parent pool, coefficients, loads and the solved level to `path`."""
        check(lib.mch_checkpoint_save(self.ctx, os.fsencode(path)), self.ctx)

    def load_checkpoint(self, path):
        """mch_checkpoint_load into a context of the same parameters and medium; solve_all()
        then continues at the next level."""
        solved = ctypes.c_int32()
        check(lib.mch_checkpoint_load(self.ctx, os.fsencode(path), ctypes.byref(solved)), self.ctx)
        self.solved = solved.value

    def coeffs_device_ptr(self):
        p = ctypes.c_void_p()
        check(lib.mch_coeffs_device(self.ctx, ctypes.byref(p)), self.ctx)
        return p.value

    def pool_info(self):
        p = ctypes.c_void_p()
        n = ctypes.c_int64()
        check(lib.mch_pool_info(self.ctx, ctypes.byref(p), ctypes.byref(n)), self.ctx)
        return p.value, n.value

    def pool_slot(self, mp):
        o = ctypes.c_int64()
        n = ctypes.c_int64()
        check(lib.mch_pool_slot(self.ctx, mp, ctypes.byref(o), ctypes.byref(n)), self.ctx)
        return o.value, n.value

    def linear_index(self, k):
        idx = 0
        for i in reversed(range(self.d)):
            idx = idx * self.mv + int(k[i])
        return idx

    def local_solution(self, k, rhs):
        """fine φ_p (Eq. 11) for macropoint k (tuple or linear index), shape [z][y][x] nodes"""
        mp = k if isinstance(k, (int, np.integer)) else self.linear_index(k)
        ext = (ctypes.c_int64 * 3)()
        cap = 1
        lmax = self.l + (self.eta ** (self.L - 1) // 2 if self.interp == "physical_s1" else 0)
        for _ in range(self.d):
            cap *= (2 * lmax + 1) * (self.n // self.M) + 1
        out = np.zeros(cap)
        check(lib.mch_local_solution(self.ctx, mp, rhs, out.ctypes.data, cap, ext), self.ctx)
        shape = tuple(ext[i] for i in reversed(range(self.d)))
        return out[: int(np.prod(shape))].reshape(shape).copy()

    def level_stats(self, level):
        s = MchLevelStats()
        check(lib.mch_get_level_stats(self.ctx, level, ctypes.byref(s)), self.ctx)
        return {f: getattr(s, f) for f, _ in MchLevelStats._fields_}

    def level_iterations(self, level):
        """[macropoints solved here, n_rhs] PCG iteration counts of the last solve of `level`"""
        n = self.level_stats(level)["problems"]
        buf = (ctypes.c_int32 * max(n, 1))()
        check(lib.mch_level_iterations(self.ctx, level, buf, n), self.ctx)
        return np.frombuffer(buf, dtype=np.int32, count=n).reshape(-1, self.n_rhs).copy()

    def num_macropoints_level(self, level):
        c = ctypes.c_int64()
        check(lib.mch_num_macropoints(self.ctx, level, ctypes.byref(c)), self.ctx)
        return c.value

    def level_macropoints(self, level):
        n = self.num_macropoints_level(level)
        buf = (ctypes.c_int64 * max(n, 1))()
        check(lib.mch_level_macropoints(self.ctx, level, buf, n), self.ctx)
        return [buf[i] for i in range(n)]

    def close(self):
        if self.ctx is not None and self.ctx.value:
            mch_destroy(self.ctx)
        self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


__all__ = ["Homogenizer", "mch_create", "mch_set_medium", "mch_solve_level", "mch_effective_coeffs",
           "mch_set_source", "mch_load_vectors", "mch_macro_solve", "mch_destroy", "_native"]

"""ctypes binding of include/mch.h (argument marshalling only; every step runs in libmch.so).

There is no fallback: if the CUDA library is missing or fails to load, importing this
module raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MCH_LIB") or os.path.join(_HERE, "lib", "libmch.so")

MCH_OK = 0
ERRORS = {-1: "MCH_EINVAL", -2: "MCH_EDIVISIBILITY", -3: "MCH_ERANK", -4: "MCH_ENOCONV",
          -5: "MCH_EORDER", -6: "MCH_ECUDA", -7: "MCH_ENOMEM", -8: "MCH_EPLAN", -9: "MCH_ENCCL"}

# every symbol include/mch.h declares
SYMBOLS = ["mch_create", "mch_set_medium", "mch_reset", "mch_solve_level", "mch_effective_coeffs", "mch_num_macropoints", "mch_level_macropoints",
           "mch_local_solution", "mch_get_level_stats", "mch_level_iterations", "mch_pool_info", "mch_pool_slot",
           "mch_coeffs_device", "mch_set_source", "mch_load_vectors", "mch_macro_solve", "mch_fine_solve",
           "mch_fine_block_averages", "mch_comm_id", "mch_comm_init", "mch_comm_destroy", "mch_shard_plan",
           "mch_checkpoint_save", "mch_checkpoint_load", "mch_last_error", "mch_destroy"]


class MchParams(ctypes.Structure):
    _fields_ = [("d", ctypes.c_int), ("n", ctypes.c_int64), ("num_continua", ctypes.c_int),
                ("M", ctypes.c_int64), ("levels", ctypes.c_int), ("eta", ctypes.c_int),
                ("oversample", ctypes.c_int), ("rtol", ctypes.c_double), ("max_iter", ctypes.c_int),
                ("rank", ctypes.c_int), ("world", ctypes.c_int), ("keep_all", ctypes.c_int),
                ("stream", ctypes.c_void_p), ("interp", ctypes.c_int), ("layout", ctypes.c_int),
                ("alloc", ctypes.c_void_p), ("free", ctypes.c_void_p), ("alloc_user", ctypes.c_void_p),
                ("nccl_comm", ctypes.c_void_p)]


ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)


def torch_allocator():
    """(alloc, free) C callbacks routing the library's device buffers through PyTorch's caching
    allocator.  Keep the returned objects alive as long as any context created with them."""
    import torch

    def _alloc(nbytes, stream, user):
        try:
            return torch.cuda.caching_allocator_alloc(int(nbytes), stream=int(stream or 0))
        except Exception:  # out of memory -> NULL -> MCH_ENOMEM
            return None

    def _free(ptr, stream, user):
        torch.cuda.caching_allocator_delete(int(ptr))

    return ALLOC_FN(_alloc), FREE_FN(_free)


class MchLevelStats(ctypes.Structure):
    _fields_ = [("macropoints", ctypes.c_int64), ("problems", ctypes.c_int64),
                ("iters_total", ctypes.c_int64), ("iters_max", ctypes.c_int64),
                ("unknowns_level", ctypes.c_int64), ("cells_level", ctypes.c_int64),
                ("relres_max", ctypes.c_double), ("ms_total", ctypes.c_double),
                ("ms_pcg", ctypes.c_double), ("ms_setup", ctypes.c_double),
                ("ms_gram", ctypes.c_double), ("pcg_bytes", ctypes.c_double),
                ("launches", ctypes.c_int64), ("rank_deficient", ctypes.c_int64),
                ("ms_comm", ctypes.c_double), ("bytes_comm", ctypes.c_double), ("node_iters", ctypes.c_double),
                ("ms_transport", ctypes.c_double), ("transport_units", ctypes.c_double),
                ("transport_flops", ctypes.c_double)]


class MchError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"CUDA library {LIB_PATH} is not built: run "
                          "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.POINTER
    vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    lib.mch_create.argtypes = [P(MchParams), vp, vp, i32, P(vp)]
    lib.mch_set_medium.argtypes = [vp, vp, vp, i32]
    lib.mch_solve_level.argtypes = [vp, i32]
    lib.mch_reset.argtypes = [vp]
    lib.mch_effective_coeffs.argtypes = [vp, vp, ctypes.c_size_t, i32]
    lib.mch_num_macropoints.argtypes = [vp, i32, P(i64)]
    lib.mch_level_macropoints.argtypes = [vp, i32, P(i64), ctypes.c_size_t]
    lib.mch_local_solution.argtypes = [vp, i64, i32, vp, ctypes.c_size_t, P(i64)]
    lib.mch_get_level_stats.argtypes = [vp, i32, P(MchLevelStats)]
    lib.mch_level_iterations.argtypes = [vp, i32, P(ctypes.c_int32), ctypes.c_size_t]
    lib.mch_pool_info.argtypes = [vp, P(vp), P(i64)]
    lib.mch_pool_slot.argtypes = [vp, i64, P(i64), P(i64)]
    lib.mch_coeffs_device.argtypes = [vp, P(vp)]
    lib.mch_checkpoint_save.argtypes = [vp, ctypes.c_char_p]
    lib.mch_checkpoint_load.argtypes = [vp, ctypes.c_char_p, P(i32)]
    lib.mch_set_source.argtypes = [vp, vp, i32]
    lib.mch_load_vectors.argtypes = [vp, vp, ctypes.c_size_t, i32]
    lib.mch_macro_solve.argtypes = [vp, vp, vp, i32, vp, ctypes.c_size_t, i32, dbl, i32, P(i32)]
    lib.mch_fine_solve.argtypes = [vp, vp, i32, vp, ctypes.c_size_t, i32, dbl, i32, P(i32)]
    lib.mch_fine_block_averages.argtypes = [vp, vp, i32, vp, ctypes.c_size_t, i32]
    lib.mch_comm_id.argtypes = [vp, ctypes.c_size_t]
    lib.mch_comm_init.argtypes = [P(vp), i32, i32, vp, ctypes.c_size_t]
    lib.mch_comm_destroy.argtypes = [vp]
    lib.mch_shard_plan.argtypes = [P(MchParams), i32, P(i64), ctypes.c_size_t, P(i64), P(i64), ctypes.c_size_t, P(i64)]
    lib.mch_last_error.argtypes = [vp]
    lib.mch_last_error.restype = ctypes.c_char_p
    lib.mch_destroy.argtypes = [vp]
    lib.mch_destroy.restype = None
    for name in SYMBOLS:
        if name not in ("mch_last_error", "mch_destroy"):
            getattr(lib, name).restype = i32
    return lib


lib = _load()


def check(rc, ctx=None):
    if rc != MCH_OK:
        msg = lib.mch_last_error(ctx)
        raise MchError(rc, msg.decode() if msg else "")

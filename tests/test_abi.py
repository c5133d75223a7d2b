"""C-ABI checks that need no GPU: libmch.so loads, exports every function include/mch.h declares,
and rejects invalid arguments before touching the device (error codes of mch.h)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "mch.h")


def _declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mch_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2503_01276_b200 import _native
    decl = _declared()
    assert "mch_create" in decl and "mch_solve_level" in decl and "mch_effective_coeffs" in decl
    nm = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\b(mch_[a-z_]+)\b", nm))
    missing = [s for s in decl if s not in exported]
    assert not missing, missing
    assert sorted(_native.SYMBOLS) == decl


def _create(**kw):
    from paper_2503_01276_b200._native import MchParams, lib
    d = kw.pop("d", 2)
    n = kw.pop("n", 32)
    kap = kw.pop("kappa", np.ones((n,) * d))
    ids = kw.pop("ids", np.zeros((n,) * d, dtype=np.uint8))
    p = MchParams(d=d, n=n, num_continua=kw.pop("N", 1), M=kw.pop("M", 4), levels=kw.pop("L", 1),
                  eta=kw.pop("eta", 2), oversample=kw.pop("l", 1), rtol=1e-12, max_iter=100, rank=0, world=1,
                  keep_all=0, stream=None, interp=kw.pop("interp", 0), layout=kw.pop("layout", 0))
    ctx = ctypes.c_void_p()
    rc = lib.mch_create(ctypes.byref(p), kap.ctypes.data, ids.ctypes.data, 0, ctypes.byref(ctx))
    return rc, lib.mch_last_error(None).decode()


@pytest.mark.parametrize("kw,code", [
    (dict(d=4), -1),                                  # MCH_EINVAL: d
    (dict(N=5), -1),                                  # MCH_EINVAL: N > 4
    (dict(M=5), -2),                                  # MCH_EDIVISIBILITY: M does not divide n
    (dict(n=24, M=8), -2),                            # H/(2h) not an integer (c = 3)
    (dict(n=32, M=8, L=3), -2),                       # H/(2 h eta^(L-1)) not an integer
    (dict(n=48, M=6, L=3), -2),                       # eta^(L-1) = 4 does not divide M
    (dict(n=32, M=4, L=3), -8),                       # MCH_EPLAN: T_1 = {0, 4}, no covering parent
    (dict(kappa=-np.ones((32, 32))), -1),             # kappa <= 0
    (dict(kappa=np.full((32, 32), np.nan)), -1),      # kappa not finite
    (dict(ids=np.full((32, 32), 3, dtype=np.uint8), N=2), -1),  # id >= N
    (dict(d=3, n=16, M=2, N=2, l=2), -1),             # 5^3 subcells x 2 continua > 108 constraint rows
    (dict(n=64, M=4, N=4, l=6), -1),                  # 2D banded projector: 676 rows x 60 band > smem
    (dict(interp=3), -1),                             # unknown interpolation mode
    (dict(interp=2, d=3, n=16, M=4, L=2, N=2), -1),   # physical-coordinate variant: 2D only
    (dict(interp=2, n=64, M=8, L=3, N=3), -1),        # ... and <= 108 level-1 rows (7x7x3 = 147)
    (dict(layout=2), -1),                             # unknown macropoint layout
    (dict(n=36, M=6, L=3, layout=1), -2),             # block layout: H/(2 h eta^(L-1)) = 3/4 not integer
])
def test_create_rejects_invalid_inputs(kw, code):
    rc, msg = _create(**kw)
    assert rc == code, (rc, msg)
    assert msg


def test_null_context_is_rejected():
    """Every context call returns MCH_EINVAL for a NULL context without touching the device."""
    from paper_2503_01276_b200._native import lib
    buf = np.zeros(16)
    it = ctypes.c_int(0)
    assert lib.mch_set_source(None, buf.ctypes.data, 0) == -1
    assert lib.mch_load_vectors(None, buf.ctypes.data, 16, 0) == -1
    assert lib.mch_macro_solve(None, None, None, 0, buf.ctypes.data, 16, 0, 1e-12, 0, ctypes.byref(it)) == -1
    assert lib.mch_solve_level(None, 1) == -1
    assert lib.mch_effective_coeffs(None, buf.ctypes.data, 16, 0) == -1
    assert lib.mch_set_medium(None, buf.ctypes.data, buf.ctypes.data, 0) == -1
    assert lib.mch_checkpoint_save(None, b"/tmp/x.mchckpt") == -1
    assert lib.mch_checkpoint_load(None, b"/tmp/x.mchckpt", None) == -1

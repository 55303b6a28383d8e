"""ctypes front-end of the C oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu-baseline /
``--impl reference`` leg may import this module.  It restates the reference's
Numba kernels (see ``tilu_oracle.c``; pinned bitwise against the live reference
by ``tests/test_oracle_golden.py``).  The product never imports it.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libtilu_oracle.so")
_lib = None

_P = ctypes.c_void_p
_I = ctypes.c_int
_L = ctypes.c_int64
_D = ctypes.c_double


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.oracle_rank_tables.argtypes = [_I, _P]
        L.oracle_surrogate_forward.argtypes = [_I, _P, _D, _P, _I, _I, _I, _P, _I, _P, _L, _P]
        L.oracle_surrogate_backward.argtypes = [_I, _P, _D, _P, _P, _I, _I, _I, _P, _I, _P, _L, _P]
        L.oracle_solve_into.argtypes = [_I, _P, _D, _P, _P, _I, _I, _I, _P, _I, _P, _L, _P]
        L.oracle_stencil_apply.argtypes = [_I, _P, _P, _I, _P, _P]
        L.oracle_surrogate_apply_residual.argtypes = [_I, _P, _D, _P, _I, _I, _I, _P, _P, _P]
        L.oracle_ilu_forward.argtypes = [_I, _P, _P, _P]
        L.oracle_ilu_backward.argtypes = [_I, _P, _P, _P]
        L.oracle_sweeps.argtypes = [_I, _D, _P, _P, _P, _I, _I, _I, _I, _P, _L, _P, _P, _I, _P,
                                    _I, _I, _I, _P, _P, _P, _I, _P]
        L.oracle_sweeps.restype = _I
        L.oracle_sweeps_many.argtypes = [_I, _D, _P, _P, _P, _I, _I, _I, _I, _P, _L, _P, _P, _I,
                                         _P, _P, _I, _I, _I]
        L.oracle_sweeps_many.restype = _I
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


def _c64(a, dtype=np.float64):
    return np.ascontiguousarray(a, dtype=dtype)


def rank_tables(level: int) -> np.ndarray:
    n = 2 ** level
    out = np.empty((n + 1, n + 1), dtype=np.int64)
    lib().oracle_rank_tables(n, _ptr(out))
    return out


class OracleSurrogate:
    """The arrays a reference ``SurrogateILU`` holds (surrogate.py:232-263)."""

    def __init__(self, level, lcoefs, dcoefs, variant="v1", band_ranks=None, store_rows=None):
        self.level = int(level)
        self.n = 2 ** self.level
        self.h = 1.0 / self.n
        self.rowoff = rank_tables(self.level)
        self.lcoefs = _c64(lcoefs)
        self.dcoefs = _c64(dcoefs).reshape(self.lcoefs.shape[1:])
        self.use_store = 1 if variant == "v1" else 0
        if band_ranks is None:
            band_ranks, store_rows = np.zeros(1, np.int64), np.zeros((1, 9))
        self.band_ranks = _c64(band_ranks, np.int64)
        self.store_rows = _c64(store_rows)
        self.k = tuple(self.lcoefs.shape[1:])

    def _common(self):
        return (self.n, _ptr(self.rowoff), self.h)

    def forward(self, w):
        kx1, ky1, kz1 = self.k
        lib().oracle_surrogate_forward(*self._common(), _ptr(self.lcoefs), kx1, ky1, kz1, _ptr(w),
                                       self.use_store, _ptr(self.band_ranks), len(self.band_ranks),
                                       _ptr(self.store_rows))

    def backward(self, w):
        kx1, ky1, kz1 = self.k
        lib().oracle_surrogate_backward(*self._common(), _ptr(self.lcoefs), _ptr(self.dcoefs), kx1,
                                        ky1, kz1, _ptr(w), self.use_store, _ptr(self.band_ranks),
                                        len(self.band_ranks), _ptr(self.store_rows))

    def solve_into(self, w: np.ndarray) -> None:
        assert w.dtype == np.float64 and w.flags.c_contiguous
        self.forward(w)
        self.backward(w)


def stencil_apply(level, arows, u):
    n = 2 ** level
    rowoff = rank_tables(level)
    arows = _c64(arows)
    aconst = 1 if arows.ndim == 1 or arows.shape[0] == 1 else 0
    out = np.zeros_like(u)
    lib().oracle_stencil_apply(n, _ptr(rowoff), _ptr(arows), aconst, _ptr(_c64(u)), _ptr(out))
    return out


def surrogate_apply_residual(level, acoefs, u, f):
    n = 2 ** level
    rowoff = rank_tables(level)
    acoefs = _c64(acoefs)
    w = np.zeros_like(u)
    kx1, ky1, kz1 = acoefs.shape[1:]
    lib().oracle_surrogate_apply_residual(n, _ptr(rowoff), 1.0 / n, _ptr(acoefs), kx1, ky1, kz1,
                                          _ptr(_c64(u)), _ptr(_c64(f)), _ptr(w))
    return w


def ilu_solve_into(level, factors, w):
    n = 2 ** level
    rowoff = rank_tables(level)
    factors = _c64(factors)
    lib().oracle_ilu_forward(n, _ptr(rowoff), _ptr(factors), _ptr(w))
    lib().oracle_ilu_backward(n, _ptr(rowoff), _ptr(factors), _ptr(w))


def sweeps(sur: OracleSurrogate | None, level, arows, u, f, nsweeps, *, factors=None,
           acoefs=None, return_norms=False):
    """``nsweeps`` smoothing steps r = f - A u -> w = solve(r) -> u += w, in place on u."""
    n = 2 ** level
    rowoff = rank_tables(level)
    arows = _c64(arows if arows is not None else np.zeros(15))
    aconst = 1 if arows.ndim == 1 or arows.shape[0] == 1 else 0
    if sur is None:
        sur = OracleSurrogate(level, np.zeros((7, 1, 1, 1)), np.zeros((1, 1, 1)), "v2")
    kx1, ky1, kz1 = sur.k
    ak = (0, 0, 0)
    if acoefs is not None:
        acoefs = _c64(acoefs)
        ak = acoefs.shape[1:]
    norms = np.zeros(nsweeps)
    assert u.dtype == np.float64 and u.flags.c_contiguous
    rc = lib().oracle_sweeps(n, 1.0 / n, _ptr(rowoff), _ptr(sur.lcoefs), _ptr(sur.dcoefs), kx1, ky1,
                             kz1, sur.use_store, _ptr(sur.band_ranks), len(sur.band_ranks),
                             _ptr(sur.store_rows), _ptr(arows), aconst, _ptr(acoefs), *ak,
                             _ptr(None if factors is None else _c64(factors)), _ptr(u),
                             _ptr(_c64(f)), nsweeps, _ptr(norms))
    if rc != 0:
        raise MemoryError("oracle_sweeps failed")
    return norms if return_norms else None


def sweeps_many(sur: OracleSurrogate, level, arow, u, f, nsweeps, nthreads=0) -> int:
    """Independent tets u[t], f[t] ([ntets, grid]) sharing one surrogate; OpenMP over tets."""
    n = 2 ** level
    arow = _c64(arow)
    assert u.ndim == 2 and u.flags.c_contiguous
    kx1, ky1, kz1 = sur.k
    used = lib().oracle_sweeps_many(n, 1.0 / n, _ptr(sur.rowoff), _ptr(sur.lcoefs), _ptr(sur.dcoefs),
                                    kx1, ky1, kz1, sur.use_store, _ptr(sur.band_ranks),
                                    len(sur.band_ranks), _ptr(sur.store_rows), _ptr(arow), 1, _ptr(u),
                                    _ptr(_c64(f)), u.shape[0], nsweeps, nthreads)
    if used < 0:
        raise MemoryError("oracle_sweeps_many failed")
    return used

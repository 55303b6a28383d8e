"""ctypes binding of libtilu.so (the C ABI declared in include/tilu.h).

The compute path has no fallback: if the CUDA library is missing or cannot be
loaded, every call raises ``TiluError`` (build it with ``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TILU_LIB", os.path.join(_HERE, "lib", "libtilu.so"))

TILU_OK, TILU_EINVAL, TILU_ECUDA, TILU_ENOMEM, TILU_EUNSUPPORTED, TILU_EPIVOT = range(6)
VARIANT_V1, VARIANT_V2 = 1, 2
FLAG_FAST, FLAG_SCHED_SIMPLE, FLAG_SCHED_PLANE, FLAG_SCHED_BATCH = 0x1, 0x2, 0x4, 0x8

_P = ctypes.c_void_p
_I = ctypes.c_int
_L = ctypes.c_int64
_D = ctypes.c_double


class TiluError(RuntimeError):
    def __init__(self, code: int, msg: str):
        self.code = code
        super().__init__(f"libtilu error {code}: {msg}")


class TiluDesc(ctypes.Structure):
    """Mirror of tilu_desc_t (include/tilu.h)."""

    _fields_ = [
        ("level", _I), ("kx1", _I), ("ky1", _I), ("kz1", _I), ("variant", _I),
        ("lcoefs", _P), ("dcoefs", _P), ("band_ranks", _P), ("nband", _L), ("store_rows", _P),
        ("arow", _P), ("arows_dev", _P), ("acoefs", _P), ("akx1", _I), ("aky1", _I), ("akz1", _I),
        ("factors", _P), ("flags", _I), ("sepk_tables", _P), ("sepk_c0", _D), ("sepk_w", _D),
        ("factors_dev", _P),
    ]


_lib = None
EXPORTS = (
    "tilu_plan_create", "tilu_plan_destroy", "tilu_solve_into", "tilu_surrogate_forward",
    "tilu_surrogate_backward", "tilu_residual", "tilu_stencil_apply", "tilu_sweep",
    "tilu_stored_solve_into", "tilu_stored_sweep", "tilu_factorize_stream", "tilu_last_error",
    "tilu_version", "tilu_last_launch_count", "tilu_plan_grid_size", "tilu_plan_interior_size",
    "tilu_profile_enable", "tilu_profile_reset", "tilu_profile_read", "tilu_packed_size",
    "tilu_packed_scratch_size", "tilu_pack",
    "tilu_unpack", "tilu_sweep_packed", "tilu_plane_tasks", "tilu_sepk_rows",
    "tilu_factorize_device", "tilu_gather_rows", "tilu_mg_restrict", "tilu_mg_prolong_add", "tilu_dense_mv",
    "tilu_csr_levels", "tilu_csr_residual_rows", "tilu_csr_tri_solve_blocks", "tilu_csr_matvec",
)


def lib():
    """Load libtilu.so once; raise loudly when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise TiluError(TILU_EUNSUPPORTED, f"{LIB_PATH} not built (run __graft_entry__.build())")
    L = ctypes.CDLL(LIB_PATH)
    L.tilu_plan_create.argtypes = [ctypes.POINTER(TiluDesc), ctypes.POINTER(_P)]
    L.tilu_plan_create.restype = _I
    L.tilu_plan_destroy.argtypes = [_P]
    L.tilu_plan_destroy.restype = None
    for name in ("tilu_solve_into", "tilu_surrogate_forward", "tilu_surrogate_backward",
                 "tilu_stored_solve_into"):
        getattr(L, name).argtypes = [_P, _P, _I, _P]
        getattr(L, name).restype = _I
    L.tilu_residual.argtypes = [_P, _P, _P, _P, _I, _P, _P]
    L.tilu_residual.restype = _I
    L.tilu_stencil_apply.argtypes = [_P, _P, _P, _I, _P]
    L.tilu_stencil_apply.restype = _I
    for name in ("tilu_sweep", "tilu_stored_sweep"):
        getattr(L, name).argtypes = [_P, _P, _P, _I, _I, _P, _P]
        getattr(L, name).restype = _I
    L.tilu_factorize_stream.argtypes = [_I, _P, _P, _I, _P, _I, _P, _L, _P, _D]
    L.tilu_factorize_stream.restype = _L
    L.tilu_last_error.restype = ctypes.c_char_p
    L.tilu_version.restype = _I
    L.tilu_last_launch_count.restype = _I
    L.tilu_plan_grid_size.argtypes = [_P]
    L.tilu_plan_grid_size.restype = _L
    L.tilu_plan_interior_size.argtypes = [_P]
    L.tilu_plan_interior_size.restype = _L
    for name in ("tilu_packed_size", "tilu_packed_scratch_size"):
        getattr(L, name).argtypes = [_P, _I]
        getattr(L, name).restype = _L
    for name in ("tilu_pack", "tilu_unpack"):
        getattr(L, name).argtypes = [_P, _P, _P, _I, _P]
        getattr(L, name).restype = _I
    L.tilu_sweep_packed.argtypes = [_P, _P, _P, _P, _I, _I, _P, _P]
    L.tilu_sweep_packed.restype = _I
    L.tilu_sepk_rows.argtypes = [_I, _P, _D, _D, _P]
    L.tilu_sepk_rows.restype = _I
    L.tilu_factorize_device.argtypes = [_I, _P, _P, _P, _D, _D, _P, _D, _P, _P]
    L.tilu_factorize_device.restype = _I
    L.tilu_gather_rows.argtypes = [_P, _P, _L, _P, _P]
    L.tilu_gather_rows.restype = _I
    L.tilu_mg_restrict.argtypes = [_I, _P, _P, _P]
    L.tilu_mg_restrict.restype = _I
    L.tilu_mg_prolong_add.argtypes = [_I, _P, _P, _P]
    L.tilu_mg_prolong_add.restype = _I
    L.tilu_dense_mv.argtypes = [_I, _P, _P, _P, _P]
    L.tilu_dense_mv.restype = _I
    L.tilu_csr_matvec.argtypes = [_L, _P, _P, _P, _P, _P, _I, _P]
    L.tilu_csr_matvec.restype = _I
    L.tilu_csr_levels.argtypes = [_I, _P, _P, _I, _P]
    L.tilu_csr_levels.restype = _I
    L.tilu_csr_residual_rows.argtypes = [_L, _P, _P, _P, _P, _P, _P, _P, _P]
    L.tilu_csr_residual_rows.restype = _I
    L.tilu_csr_tri_solve_blocks.argtypes = [_I, _P, _P, _P, _P, _P, _P, _P, _I, _P, _P, _P, _P, _P]
    L.tilu_csr_tri_solve_blocks.restype = _I
    L.tilu_plane_tasks.argtypes = [_I, _P, _I]
    L.tilu_plane_tasks.restype = _I
    L.tilu_profile_enable.argtypes = [_I]
    L.tilu_profile_enable.restype = None
    L.tilu_profile_reset.restype = None
    L.tilu_profile_read.argtypes = [_P, _P, _P, _I]
    L.tilu_profile_read.restype = _I
    _lib = L
    return L


def check(rc: int) -> None:
    if rc != TILU_OK:
        raise TiluError(rc, lib().tilu_last_error().decode(errors="replace"))


def last_launch_count() -> int:
    return int(lib().tilu_last_launch_count())


def profile_enable(on: bool = True) -> None:
    lib().tilu_profile_enable(1 if on else 0)
    lib().tilu_profile_reset()


def profile_read() -> dict:
    """{kernel family: (launches, total ms)} of the kernels launched while profiling was on."""
    cap = 64
    names = ctypes.create_string_buffer(64 * cap)
    counts = (ctypes.c_int * cap)()
    ms = (ctypes.c_double * cap)()
    k = lib().tilu_profile_read(names, counts, ms, cap)
    out = {}
    for i in range(min(k, cap)):
        nm = names.raw[64 * i:64 * (i + 1)].split(b"\0", 1)[0].decode()
        out[nm] = (int(counts[i]), float(ms[i]))
    return out


def plane_tasks(level: int) -> list[tuple[int, int]]:
    """(band, chunk) tasks of the single-tet plane kernels in forward topological order."""
    L = lib()
    n = int(L.tilu_plane_tasks(int(level), None, 0))
    buf = (ctypes.c_int * max(n, 1))()
    L.tilu_plane_tasks(int(level), buf, n)
    return [(v >> 16, v & 0xFFFF) for v in buf[:n]]

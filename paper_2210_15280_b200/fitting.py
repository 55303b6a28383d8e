"""Host-side setup of the surrogate ILU(0): streaming factorization, strided sampling,
least-squares fit of the factor stencil fields (arXiv 2210.15280, Alg. 1 + Sec. 4.1).

This is the setup that stays on the host (BASELINE north_star).  The factorization
runs in native code (``tilu_factorize_stream`` in libtilu, a restatement of
reference _kernels.py:39-143); sampling and the fit follow the reference recipe
(surrogate.py:68-337) with the same numpy/LAPACK primitives so the fitted
coefficient tables are bitwise identical to the reference's when BLAS runs on one
thread (tests/test_setup_parity.py).  Only the evaluation of those tables, i.e. the
smoothing sweep, runs on the GPU (smoother.py).
"""

from __future__ import annotations

import contextlib
import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib, lattice
from .stencil import StencilSource


class RankDeficientFit(RuntimeError):
    pass


class EmptySampleSet(RuntimeError):
    pass


class PivotBreakdown(RuntimeError):
    def __init__(self, coord):
        self.coord = tuple(int(c) for c in coord)
        super().__init__(f"zero pivot at logical coordinate {self.coord}")


@contextlib.contextmanager
def single_thread_blas():
    """The LAPACK least-squares solution depends on the BLAS thread count;
    the reference's setup is reproduced with one thread."""
    try:
        from threadpoolctl import threadpool_limits
    except ImportError:  # pragma: no cover - threadpoolctl ships in this image
        yield
        return
    with threadpool_limits(limits=1, user_api="blas"):
        yield


# ------------------------------------------------------------------------------------------
# polynomials
# ------------------------------------------------------------------------------------------

def design_matrix(points: np.ndarray, degrees) -> np.ndarray:
    """Monomials X^i Y^j Z^k, ravelled (i, j, k) C-order (reference surrogate.py:68-73)."""
    dgx, dgy, dgz = degrees
    px = points[:, 0][:, None] ** np.arange(dgx + 1)
    py = points[:, 1][:, None] ** np.arange(dgy + 1)
    pz = points[:, 2][:, None] ** np.arange(dgz + 1)
    return np.einsum("mi,mj,mk->mijk", px, py, pz).reshape(len(points), -1)


@dataclass
class SurrogatePolynomial:
    """sum c[i,j,k] X^i Y^j Z^k with X = x*h etc. (logical coordinates scaled by h)."""

    degrees: tuple
    coef: np.ndarray
    spacing: float

    def evaluate_scaled(self, points) -> np.ndarray:
        points = np.atleast_2d(np.asarray(points, dtype=np.float64))
        return design_matrix(points, self.degrees) @ self.coef.ravel()

    def evaluate_logical(self, coords) -> np.ndarray:
        return self.evaluate_scaled(np.asarray(coords, dtype=np.float64) * self.spacing)

    @classmethod
    def zero(cls, degrees, spacing) -> "SurrogatePolynomial":
        return cls(tuple(degrees), np.zeros(tuple(d + 1 for d in degrees)), spacing)


def lsq_fit(points, values, degrees, spacing: float = 1.0, label: str = "") -> SurrogatePolynomial:
    """Monomial least squares by orthogonal factorization (LAPACK gelsd via numpy)."""
    degrees = tuple(int(d) for d in degrees)
    M = design_matrix(np.atleast_2d(np.asarray(points, dtype=np.float64)), degrees)
    what = f" for {label}" if label else ""
    if M.shape[0] < M.shape[1]:
        raise RankDeficientFit(f"underdetermined fit{what}")
    sol, _, rank, _ = np.linalg.lstsq(M, np.asarray(values, dtype=np.float64), rcond=None)
    if rank < M.shape[1]:
        raise RankDeficientFit(f"rank-deficient design matrix{what}")
    return SurrogatePolynomial(degrees, sol.reshape(tuple(d + 1 for d in degrees)), spacing)


def nddf_row_evaluate(poly: SurrogatePolynomial, start, count: int) -> np.ndarray:
    """Values along an x-row by forward differences seeded from direct evaluation
    (reference surrogate.py:93-117; host helper, not the kernels' seeding)."""
    if count <= 0:
        return np.empty(0)
    x0, y0, z0 = (int(c) for c in start)
    h = poly.spacing
    seed = min(poly.degrees[0] + 1, count)
    pts = np.stack([(x0 + np.arange(seed)) * h, np.full(seed, y0 * h), np.full(seed, z0 * h)], axis=1)
    table = poly.evaluate_scaled(pts)
    for order in range(1, seed):
        table[order:] = table[order:] - table[order - 1:-1].copy()
    out = np.empty(count)
    for t in range(count):
        out[t] = table[0]
        for j in range(seed - 1):
            table[j] += table[j + 1]
    return out


# ------------------------------------------------------------------------------------------
# sampling
# ------------------------------------------------------------------------------------------

def sample_coords(d: int, level: int, stride: int) -> np.ndarray:
    """Sample set S_d: interior p = (1 - d) + stride * k with p + d interior, sorted (z, y, x)."""
    n = 2 ** level
    off = lattice.OFFSETS[d]
    start = 1 - off
    ax = [np.arange(start[a], n + 1, stride) for a in range(3)]
    gx, gy, gz = np.meshgrid(*ax, indexing="ij")
    pts = np.stack([gx.ravel(), gy.ravel(), gz.ravel()], axis=1)
    pts = pts[lattice.is_interior(pts, level)]
    if len(pts):
        pts = pts[lattice.is_interior(pts + off, level)]
    if len(pts):
        pts = pts[np.lexsort((pts[:, 0], pts[:, 1], pts[:, 2]))]
    return pts


def supported_degrees(coord_sets, degrees) -> tuple:
    """Clamp degrees to what the sample sets resolve (distinct values per axis, #samples)."""
    eff = list(degrees)
    nonempty = [c for c in coord_sets if len(c)]
    for coords in nonempty:
        for a in range(3):
            eff[a] = min(eff[a], len(np.unique(coords[:, a])) - 1)
    eff = [max(0, e) for e in eff]
    min_count = min(len(c) for c in nonempty) if nonempty else 1
    while (eff[0] + 1) * (eff[1] + 1) * (eff[2] + 1) > min_count:
        j = int(np.argmax(eff))
        if eff[j] == 0:
            break
        eff[j] -= 1
    return tuple(eff)


def choose_stride(level: int, sample_level, degrees, directions) -> int:
    """Largest power-of-two stride (from the sampling level, default L-2 clamped to >= 2)
    whose sample sets still resolve the requested degrees."""
    lh = max(2, level - 2) if sample_level is None else max(2, min(sample_level, level))
    stride = 2 ** (level - lh)
    while stride > 1:
        sets = [sample_coords(d, level, stride) for d in directions]
        if all(len(s) for s in sets) and supported_degrees(sets, degrees) == tuple(degrees):
            break
        stride //= 2
    return stride


def fit_with_degrade(fit_all, degrees):
    """Fit; on rank deficiency lower the largest degree of all targets jointly and retry."""
    deg = tuple(degrees)
    while True:
        try:
            return fit_all(deg), deg
        except RankDeficientFit:
            if max(deg) == 0:
                raise
            j = int(np.argmax(deg))
            deg = tuple(d - 1 if a == j else d for a, d in enumerate(deg))


def inverse_diag_positive(poly: SurrogatePolynomial, level: int, variant: str, chunk: int = 1 << 20) -> bool:
    """Is the fitted 1/D positive wherever the sweep evaluates it (outside the V1 band)?
    Evaluated in z-slabs so level 9 does not materialise a 22 GB design matrix."""
    coords = lattice.lattice_coords(level, "interior")
    if variant == "v1":
        coords = coords[~lattice.band_mask(coords, level)]
    if len(coords) == 0:
        return True
    lo = np.inf
    for s in range(0, len(coords), chunk):
        lo = min(lo, float(poly.evaluate_logical(coords[s:s + chunk]).min()))
    return bool(lo > 0.0)


# ------------------------------------------------------------------------------------------
# factorization (native)
# ------------------------------------------------------------------------------------------

@dataclass
class FactorizationResult:
    level: int
    rows: np.ndarray | None        # [grid, 9] full store (L_w..L_be, D, 1/D) or None
    collected: np.ndarray | None   # [len(collect_ranks), 9]
    aux_bytes: int
    store_bytes: int


def _pivot_eps(source: StencilSource) -> float:
    if source.data is None and source.sepk is not None:
        # table-form source without materialised rows: bound of the centre entry (<= 24 k W)
        t = np.abs(np.asarray(source.sepk.tables))
        kmax = abs(float(source.sepk.c0)) + float(t[0].max() * t[1].max() * t[2].max())
        return 1e-300 * max(24.0 * kmax * float(source.sepk.w), 1.0)
    data = np.atleast_2d(source.data)
    scale = abs(float(data[0, lattice.C])) if source.constant else float(np.abs(data[:, lattice.C]).max())
    return 1e-300 * max(scale, 1.0)


def factorize_tet(source: StencilSource, level: int, *, full_store: bool = True,
                  collect_ranks=None) -> FactorizationResult:
    """Streaming LDL^T ILU(0) of one macro-tet interior (native two-layer sweep)."""
    n = 2 ** level
    rowoff = np.ascontiguousarray(lattice.rank_tables(level))
    arows, aconst = source.kernel_args
    arows = np.ascontiguousarray(arows, dtype=np.float64)
    cr = np.ascontiguousarray(np.empty(0, np.int64) if collect_ranks is None else collect_ranks, dtype=np.int64)
    collected = np.zeros((len(cr), 9))
    rows = np.zeros((lattice.grid_size(level), 9)) if full_store else np.zeros((1, 9))
    status = _lib.lib().tilu_factorize_stream(
        n, rowoff.ctypes.data, arows.ctypes.data, int(bool(aconst)), rows.ctypes.data, int(full_store),
        cr.ctypes.data, len(cr), collected.ctypes.data, ctypes.c_double(_pivot_eps(source)))
    if status != 0:
        raise PivotBreakdown(lattice.lattice_coords(level)[status - 1])
    tri = (n + 1) * (n + 2) // 2
    return FactorizationResult(level, rows if full_store else None, collected if len(cr) else None,
                               2 * tri * 8 * 8 + collected.nbytes, rows.nbytes if full_store else 0)


def factorize_tet_device(source: StencilSource, level: int, *, full_store: bool = True, collect_ranks=None,
                         device="cuda", keep_on_device: bool = False) -> FactorizationResult:
    """The same factorization on the GPU (``tilu_factorize_device``: hyperplane-wavefront kernel, bitwise
    equal to ``factorize_tet`` / the reference's ``factorize_stream``).  The operator comes from the
    source's cheapest form: the separable-coefficient tables (config 3: rows evaluated on the fly, no
    [grid, 15] array), the constant row, or the per-point rows (uploaded).  ``collect_ranks`` rows are
    gathered on the device and returned as a host array; the full store is returned as a host array, or
    as the CUDA tensor itself with ``keep_on_device`` (for ``DevicePlan(factors=...)``)."""
    import torch

    L = _lib.lib()
    dev = torch.device(device)
    grid = lattice.grid_size(level)
    with torch.cuda.device(dev):
        store = torch.zeros((grid, 9), dtype=torch.float64, device=dev)
        status = ctypes.c_int64(0)
        stream = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
        rows_dev = tab_dev = None
        arow = None
        c0 = w = 0.0
        if getattr(source, "sepk", None) is not None:
            tab_dev = torch.as_tensor(np.ascontiguousarray(source.sepk.tables, dtype=np.float64), device=dev)
            c0, w = float(source.sepk.c0), float(source.sepk.w)
        elif source.constant:
            arow = np.ascontiguousarray(np.atleast_1d(source.data), dtype=np.float64).reshape(15)
        else:
            data = source.data
            rows_dev = (data if isinstance(data, torch.Tensor) else
                        torch.as_tensor(np.ascontiguousarray(data, dtype=np.float64), device=dev)).contiguous()
            if tuple(rows_dev.shape) != (grid, 15) or rows_dev.dtype != torch.float64 or not rows_dev.is_cuda:
                raise ValueError(f"per-point operator rows must be float64 [{grid}, 15] on the device")
        rc = L.tilu_factorize_device(
            level, rows_dev.data_ptr() if rows_dev is not None else None,
            arow.ctypes.data if arow is not None else None,
            tab_dev.data_ptr() if tab_dev is not None else None, ctypes.c_double(c0), ctypes.c_double(w),
            store.data_ptr(), ctypes.c_double(_pivot_eps(source)), ctypes.byref(status), stream)
        if rc == _lib.TILU_EPIVOT:
            raise PivotBreakdown(lattice.lattice_coords(level)[status.value - 1])
        _lib.check(rc)
        collected = None
        if collect_ranks is not None and len(collect_ranks):
            cr = torch.as_tensor(np.ascontiguousarray(collect_ranks, dtype=np.int64), device=dev)
            out = torch.empty((len(cr), 9), dtype=torch.float64, device=dev)
            _lib.check(L.tilu_gather_rows(store.data_ptr(), cr.data_ptr(), len(cr), out.data_ptr(), stream))
            collected = out.cpu().numpy()
        rows = None
        if full_store:
            rows = store if keep_on_device else store.cpu().numpy()
    return FactorizationResult(level, rows, collected, 0 if collected is None else collected.nbytes,
                               grid * 72 if full_store else 0)


# ------------------------------------------------------------------------------------------
# the surrogate build (Alg. 1 sampling + 8 least-squares problems)
# ------------------------------------------------------------------------------------------

@dataclass
class SurrogateFit:
    """Everything a reference SurrogateILU holds (surrogate.py:232-252)."""

    level: int
    degrees: tuple            # effective degrees after degrade
    variant: str
    polys: dict               # direction name -> SurrogatePolynomial, plus 'inv_dc'
    band_ranks: np.ndarray
    store_rows: np.ndarray
    sample_level: int
    stride: int
    aux_bytes: int

    @property
    def lcoefs(self) -> np.ndarray:
        return np.stack([self.polys[lattice.DIRECTION_NAMES[d]].coef for d in lattice.LOWER])

    @property
    def dcoefs(self) -> np.ndarray:
        return self.polys["inv_dc"].coef[None]


def fit_surrogate_ilu(source: StencilSource, level: int, degrees, variant: str = "v1",
                      sample_level=None, factorize: str = "host") -> SurrogateFit:
    """``factorize``: "host" (native two-layer sweep on the CPU) or "device" (the wavefront kernel on the
    GPU; same factor rows bitwise, so the fit is identical)."""
    if factorize not in ("host", "device"):
        raise ValueError(f"unknown factorize mode {factorize!r}")
    if variant not in ("v1", "v2"):
        raise ValueError(f"unknown variant {variant!r}")
    degrees = tuple(int(d) for d in degrees)
    targets = list(lattice.LOWER) + [lattice.C]
    stride = choose_stride(level, sample_level, degrees, targets)
    band = lattice.band_ranks(level) if variant == "v1" else np.empty(0, dtype=np.int64)
    h = 1.0 / 2 ** level
    with single_thread_blas():
        while True:
            sets = {}
            for d in targets:
                coords = sample_coords(d, level, stride)
                if len(coords) == 0 and level > 2:
                    raise EmptySampleSet(f"empty sample set for direction {lattice.DIRECTION_NAMES[d]!r}")
                sets[d] = coords
            eff = supported_degrees([sets[d] for d in targets], degrees)
            ranks = [lattice.lattice_rank(c, level) for c in sets.values() if len(c)]
            union = np.unique(np.concatenate(ranks + [band]))
            res = (factorize_tet_device if factorize == "device" else factorize_tet)(
                source, level, full_store=False, collect_ranks=union)
            rows = res.collected

            def fit_all(deg, sets=sets, union=union, rows=rows):
                polys = {}
                for slot, d in enumerate(lattice.LOWER):
                    name = lattice.DIRECTION_NAMES[d]
                    coords = sets[d]
                    if len(coords) == 0:
                        polys[name] = SurrogatePolynomial.zero(deg, h)
                        continue
                    vals = rows[np.searchsorted(union, lattice.lattice_rank(coords, level)), slot]
                    polys[name] = lsq_fit(coords * h, vals, deg, spacing=h, label=name)
                coords = sets[lattice.C]
                vals = rows[np.searchsorted(union, lattice.lattice_rank(coords, level)), 8]
                polys["inv_dc"] = lsq_fit(coords * h, vals, deg, spacing=h, label="inv_dc")
                return polys

            polys, eff = fit_with_degrade(fit_all, eff)
            if stride == 1 or inverse_diag_positive(polys["inv_dc"], level, variant):
                break
            stride //= 2   # fitted 1/D dipped non-positive: densify the samples and refit
    if variant == "v1":
        store_rows = rows[np.searchsorted(union, band)].copy()
    else:
        store_rows, band = np.zeros((1, 9)), np.zeros(1, dtype=np.int64)
    return SurrogateFit(level, eff, variant, polys, band, store_rows, level - int(np.log2(stride)), stride,
                        res.aux_bytes + store_rows.nbytes + band.nbytes)


def fit_surrogate_operator(source: StencilSource, level: int, degrees, sample_level=None) -> np.ndarray:
    """Coefficient tables [15][kx+1][ky+1][kz+1] of the operator surrogate
    (reference surrogate.py:361-388); used by a_mode='surrogate'."""
    degrees = tuple(int(d) for d in degrees)
    dirs = list(range(15))
    stride = choose_stride(level, sample_level, degrees, dirs)
    h = 1.0 / 2 ** level
    sets = {d: sample_coords(d, level, stride) for d in dirs}
    eff = supported_degrees(list(sets.values()), degrees)

    def fit_all(deg):
        out = {}
        for d in dirs:
            coords = sets[d]
            if len(coords) == 0:
                if level > 2:
                    raise EmptySampleSet(f"empty sample set for direction {lattice.DIRECTION_NAMES[d]!r}")
                coords = lattice.lattice_coords(level, "interior")
            if source.constant:
                vals = np.full(len(coords), np.atleast_1d(source.data)[d])
            else:
                vals = source.data[lattice.lattice_rank(coords, level), d]
            out[d] = lsq_fit(coords * h, vals, deg, spacing=h, label=lattice.DIRECTION_NAMES[d])
        return out

    with single_thread_blas():
        polys, _ = fit_with_degrade(fit_all, eff)
    return np.stack([polys[d].coef for d in dirs])

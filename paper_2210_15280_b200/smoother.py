"""Device-side smoother objects: the drop-in boundary of the hot path.

Mirrors the reference's cell-preconditioner protocol (duck-typed ``solve_into(w)``,
surrogate.py:258, ilu.py:225) and adds the north-star ``apply(u, f, sweeps)``.
All compute goes through libtilu's C ABI (include/tilu.h); there is no CPU
fallback -- a missing library or a CPU tensor raises.

Vectors are fp64 in the reference's full-lattice rank layout, zero outside the
interior, either one macro-tet ``[grid]`` or a batch ``[ntets, grid]`` of tets that
share one surrogate (identical operator, e.g. the Kuhn tets of config 4).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib, fitting, lattice
from .stencil import CoefficientField, StencilSource, stencil_source

try:  # torch provides device memory and streams (plumbing only)
    import torch
except ImportError:  # pragma: no cover
    torch = None


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _stream_ptr():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _as_batch(t, grid: int, name: str):
    """Validate a CUDA fp64 contiguous tensor of shape [grid] or [T, grid]; return (tensor, T)."""
    if torch is None or not isinstance(t, torch.Tensor):
        raise TypeError(f"{name}: expected a torch.Tensor on a CUDA device")
    if not t.is_cuda:
        raise ValueError(f"{name}: tensor must live on a CUDA device (no CPU fallback)")
    if t.dtype != torch.float64:
        raise TypeError(f"{name}: dtype must be float64, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name}: tensor must be contiguous")
    if t.shape[-1] != grid or t.dim() not in (1, 2):
        raise ValueError(f"{name}: expected shape [{grid}] or [ntets, {grid}], got {tuple(t.shape)}")
    return t, (1 if t.dim() == 1 else t.shape[0])


def _same_batch(ref, T: int, grid: int, **others):
    """Every tensor in ``others`` must be a CUDA fp64 batch of exactly ``ref``'s shape on ``ref``'s
    device: the kernels read ``T * grid`` doubles from each of them."""
    out = []
    for name, t in others.items():
        t, Tn = _as_batch(t, grid, name)
        if tuple(t.shape) != tuple(ref.shape) or Tn != T:
            raise ValueError(f"{name}: shape {tuple(t.shape)} does not match u's {tuple(ref.shape)}")
        if t.device != ref.device:
            raise ValueError(f"{name}: on {t.device}, u on {ref.device}")
        out.append(t)
    return out


class DevicePlan:
    """Owner of one ``tilu_plan_t`` (coefficients, band rows, operator and seed tables on device)."""

    def __init__(self, level: int, lcoefs, dcoefs, variant: str = "v1", band_ranks=None, store_rows=None,
                 arow=None, arows=None, acoefs=None, factors=None, fast: bool = False, simple: bool = False,
                 schedule: str = "auto", sepk=None):
        """schedule: "auto" (single tets: plane kernels from level 5, batches: interleaved kernels),
        "simple" (reference-layout wavefront kernels), "plane" (plane kernels at every level),
        "batch" (interleaved dataflow kernels for single tets too).
        sepk: a stencil.SeparableK -- the residual evaluates the separable coefficient's rows on the
        fly (config 3) instead of reading arow / arows."""
        L = _lib.lib()
        self.level = int(level)
        self.variant = variant
        self._keep = []
        lcoefs = _f64(lcoefs)
        if lcoefs.ndim != 4 or lcoefs.shape[0] != 7:
            raise ValueError("lcoefs must be [7, kx+1, ky+1, kz+1]")
        dcoefs = _f64(dcoefs).reshape(lcoefs.shape[1:])
        d = _lib.TiluDesc()
        d.level = self.level
        d.kx1, d.ky1, d.kz1 = lcoefs.shape[1:]
        d.variant = _lib.VARIANT_V1 if variant == "v1" else _lib.VARIANT_V2
        d.lcoefs, d.dcoefs = self._ptr(lcoefs), self._ptr(dcoefs)
        if variant == "v1":
            br, sr = np.ascontiguousarray(band_ranks, dtype=np.int64), _f64(store_rows)
            d.band_ranks, d.nband, d.store_rows = self._ptr(br), len(br), self._ptr(sr)
        if arow is not None:
            d.arow = self._ptr(_f64(arow).reshape(15))
        if arows is not None:
            if not (isinstance(arows, torch.Tensor) and arows.is_cuda and arows.dtype == torch.float64):
                arows = torch.as_tensor(_f64(arows), device="cuda")
            self._arows = arows.contiguous()
            d.arows_dev = self._arows.data_ptr()
        if acoefs is not None:
            ac = _f64(acoefs)
            d.acoefs = self._ptr(ac)
            d.akx1, d.aky1, d.akz1 = ac.shape[1:]
        if isinstance(factors, torch.Tensor) and factors.is_cuda:
            # device-resident factor store (fitting.factorize_tet_device): used in place, no upload
            if factors.dtype != torch.float64 or not factors.is_contiguous():
                raise ValueError("device factors must be a contiguous float64 tensor [grid, 9]")
            self._factors = factors
            d.factors_dev = factors.data_ptr()
        elif factors is not None:
            d.factors = self._ptr(_f64(factors))
        if sepk is not None:
            if int(sepk.level) != self.level:
                raise ValueError(f"sepk tables are for level {sepk.level}, plan level {self.level}")
            tab = _f64(sepk.tables)
            if tab.shape != (3, 4 * 2 ** self.level + 1):
                raise ValueError("sepk tables must be [3, 4n+1]")
            d.sepk_tables, d.sepk_c0, d.sepk_w = self._ptr(tab), float(sepk.c0), float(sepk.w)
        if schedule not in ("auto", "simple", "plane", "batch"):
            raise ValueError(f"unknown schedule {schedule!r}")
        simple = simple or schedule == "simple"
        d.flags = ((_lib.FLAG_FAST if fast else 0) | (_lib.FLAG_SCHED_SIMPLE if simple else 0)
                   | (_lib.FLAG_SCHED_PLANE if schedule == "plane" else 0)
                   | (_lib.FLAG_SCHED_BATCH if schedule == "batch" else 0))
        self.fast = fast
        handle = ctypes.c_void_p()
        _lib.check(L.tilu_plan_create(ctypes.byref(d), ctypes.byref(handle)))
        self._h = handle
        self._keep.clear()
        self.grid = int(L.tilu_plan_grid_size(handle))
        self.interior = int(L.tilu_plan_interior_size(handle))
        self.kx1 = int(lcoefs.shape[1])

    def _ptr(self, a: np.ndarray):
        self._keep.append(a)
        return a.ctypes.data

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _lib.lib().tilu_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    # -- calls ------------------------------------------------------------------------------
    def solve_into(self, w) -> None:
        w, T = _as_batch(w, self.grid, "w")
        _lib.check(_lib.lib().tilu_solve_into(self._h, w.data_ptr(), T, _stream_ptr()))

    def forward(self, w) -> None:
        w, T = _as_batch(w, self.grid, "w")
        _lib.check(_lib.lib().tilu_surrogate_forward(self._h, w.data_ptr(), T, _stream_ptr()))

    def backward(self, w) -> None:
        w, T = _as_batch(w, self.grid, "w")
        _lib.check(_lib.lib().tilu_surrogate_backward(self._h, w.data_ptr(), T, _stream_ptr()))

    def stored_solve_into(self, w) -> None:
        w, T = _as_batch(w, self.grid, "w")
        _lib.check(_lib.lib().tilu_stored_solve_into(self._h, w.data_ptr(), T, _stream_ptr()))

    def residual(self, u, f, w=None, norms: bool = False):
        u, T = _as_batch(u, self.grid, "u")
        if w is None:
            w = torch.zeros_like(u)
        f, w = _same_batch(u, T, self.grid, f=f, w=w)
        rn = torch.empty(T, dtype=torch.float64, device=u.device) if norms else None
        _lib.check(_lib.lib().tilu_residual(self._h, u.data_ptr(), f.data_ptr(), w.data_ptr(), T,
                                            None if rn is None else rn.data_ptr(), _stream_ptr()))
        return (w, rn) if norms else w

    def stencil_apply(self, u, out=None):
        u, T = _as_batch(u, self.grid, "u")
        if out is None:
            out = torch.zeros_like(u)
        (out,) = _same_batch(u, T, self.grid, out=out)
        _lib.check(_lib.lib().tilu_stencil_apply(self._h, u.data_ptr(), out.data_ptr(), T, _stream_ptr()))
        return out

    def sweep(self, u, f, sweeps: int = 1, norms: bool = False, stored: bool = False):
        """``sweeps`` smoothing steps in place on u; returns ||f - A u||^2 before each sweep
        ([sweeps, ntets]) when ``norms``."""
        u, T = _as_batch(u, self.grid, "u")
        (f,) = _same_batch(u, T, self.grid, f=f)
        rn = torch.empty((sweeps, T), dtype=torch.float64, device=u.device) if norms else None
        fn = _lib.lib().tilu_stored_sweep if stored else _lib.lib().tilu_sweep
        _lib.check(fn(self._h, u.data_ptr(), f.data_ptr(), T, int(sweeps),
                      None if rn is None else rn.data_ptr(), _stream_ptr()))
        return rn

    # -- packed (interleaved) batches: resident state for many tets sharing this plan ----------
    def packed_numel(self, ntets: int) -> int:
        return int(_lib.lib().tilu_packed_size(self._h, int(ntets)))

    def scratch_numel(self, ntets: int) -> int:
        return int(_lib.lib().tilu_packed_scratch_size(self._h, int(ntets)))

    def new_scratch(self, ntets: int, device="cuda"):
        """Zeroed scratch for :meth:`sweep_packed` (keeps its own state across calls; reuse it only
        with this plan and the same ntets)."""
        return torch.zeros(self.scratch_numel(ntets), dtype=torch.float64, device=device)

    def pack(self, src, ntets: int | None = None, out=None):
        src, T = _as_batch(src, self.grid, "src")
        if ntets is not None:
            if not 1 <= int(ntets) <= T:
                raise ValueError(f"ntets={ntets}: src holds {T} tets")
            T = int(ntets)
        if out is None:
            out = torch.empty(self.packed_numel(T), dtype=torch.float64, device=src.device)
        _lib.check(_lib.lib().tilu_pack(self._h, src.data_ptr(), out.data_ptr(), T, _stream_ptr()))
        return out

    def unpack(self, src, out):
        out, T = _as_batch(out, self.grid, "out")
        if src.numel() != self.packed_numel(T):
            raise ValueError("packed buffer size does not match ntets")
        _lib.check(_lib.lib().tilu_unpack(self._h, src.data_ptr(), out.data_ptr(), T, _stream_ptr()))
        return out

    def sweep_packed(self, u_p, f_p, w_p, ntets: int, sweeps: int = 1, norms: bool = False):
        """Fused sweeps on packed u, f (w_p: scratch from :meth:`new_scratch`)."""
        for name, t, size in (("u_p", u_p, self.packed_numel(ntets)), ("f_p", f_p, self.packed_numel(ntets)),
                              ("w_p", w_p, self.scratch_numel(ntets))):
            if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous() and t.numel() == size):
                raise ValueError(f"{name}: CUDA fp64 buffer of {size} doubles required")
        rn = torch.empty((sweeps, ntets), dtype=torch.float64, device=u_p.device) if norms else None
        _lib.check(_lib.lib().tilu_sweep_packed(self._h, u_p.data_ptr(), f_p.data_ptr(), w_p.data_ptr(), int(ntets),
                                                int(sweeps), None if rn is None else rn.data_ptr(), _stream_ptr()))
        return rn

    @staticmethod
    def last_launch_count() -> int:
        return _lib.last_launch_count()


def _device_solve_into(plan_fn, grid: int, w) -> None:
    """solve_into on a CUDA tensor (in place) or, for dropping into the reference's host code,
    on a numpy vector (copied to the device and back)."""
    if isinstance(w, np.ndarray):
        if w.dtype != np.float64 or w.shape[-1] != grid:
            raise ValueError(f"w must be float64 [..., {grid}]")
        t = torch.as_tensor(np.ascontiguousarray(w), device="cuda")
        plan_fn(t)
        w[...] = t.cpu().numpy()
        return
    plan_fn(w)


class SurrogateILU(fitting.SurrogateFit):
    """Polynomial surrogate of the ILU(0) factor fields of one cell (reference
    surrogate.py:232-263); ``solve_into`` runs on the GPU."""

    def __init__(self, fit: fitting.SurrogateFit, fast: bool = False):
        super().__init__(**fit.__dict__)
        self._fast = fast
        self._plan = None

    @property
    def use_store(self) -> bool:
        return self.variant == "v1"

    @property
    def _lcoefs(self):
        return self.lcoefs

    @property
    def _dcoefs(self):
        return self.dcoefs

    @property
    def _band_ranks(self):
        return self.band_ranks

    @property
    def _store_rows(self):
        return self.store_rows

    def plan(self, **op) -> DevicePlan:
        if op:
            return DevicePlan(self.level, self.lcoefs, self.dcoefs, self.variant, self.band_ranks,
                              self.store_rows, fast=self._fast, **op)
        if self._plan is None:
            self._plan = DevicePlan(self.level, self.lcoefs, self.dcoefs, self.variant, self.band_ranks,
                                    self.store_rows, fast=self._fast)
        return self._plan

    def solve_into(self, w) -> None:
        _device_solve_into(self.plan().solve_into, lattice.grid_size(self.level), w)


def build_surrogate_ilu(source: StencilSource, level: int, degrees, variant: str = "v1",
                        sample_level=None, fast: bool = False, factorize: str = "host") -> SurrogateILU:
    """Setup (streaming factorization + LSQ fit) of a device surrogate ILU(0) (reference
    surrogate.py:266-326); ``factorize="device"`` runs the factorization sweep on the GPU (same rows
    bitwise), the least-squares fit stays on the host."""
    return SurrogateILU(fitting.fit_surrogate_ilu(source, level, degrees, variant, sample_level, factorize), fast)


class CellILU:
    """Stored-factor ILU(0) of one cell (reference ilu.py:210-227) on the GPU: the
    comparison sweep for configs 1 and 5."""

    def __init__(self, result: fitting.FactorizationResult):
        if result.rows is None:
            raise ValueError("CellILU needs a full factor store")
        self.level = result.level
        self.rows = result.rows
        self._plan = None

    def plan(self, **op) -> DevicePlan:
        z = np.zeros((7, 1, 1, 1))
        if op:
            return DevicePlan(self.level, z, np.zeros(1), "v2", factors=self.rows, **op)
        if self._plan is None:
            self._plan = DevicePlan(self.level, z, np.zeros(1), "v2", factors=self.rows)
        return self._plan

    def solve_into(self, w) -> None:
        _device_solve_into(self.plan().stored_solve_into, lattice.grid_size(self.level), w)


@dataclass(frozen=True)
class SmootherConfig:
    """Smoother knobs (reference multigrid.py:39-70); this library implements the
    'surrogate_ilu' and 'ilu' kinds on the GPU."""

    kind: str = "surrogate_ilu"
    degrees: tuple = (3, 3, 3)
    variant: str = "v1"
    sample_level: int | None = None
    a_mode: str = "assembled"
    a_degrees: tuple = (3, 3, 3)

    def __post_init__(self):
        if self.kind not in ("ilu", "surrogate_ilu"):
            raise ValueError(f"unsupported smoother kind {self.kind!r} (GPU path: 'ilu', 'surrogate_ilu')")
        if self.variant not in ("v1", "v2"):
            raise ValueError(f"unknown variant {self.variant!r}")
        if self.a_mode not in ("assembled", "surrogate"):
            raise ValueError(f"unknown a_mode {self.a_mode!r}")


class SurrogateILUSmoother:
    """The north-star API: setup from the operator, level and degree, then
    ``apply(u, f, sweeps)`` = ``sweeps`` single-tet all-Dirichlet cell stages
    (multigrid.py:414-429) on the GPU."""

    def __init__(self, source: StencilSource, level: int, config: SmootherConfig, fast: bool = False,
                 simple: bool = False, factorize: str = "host"):
        self.source = source
        self.level = level
        self.config = config
        self.grid = lattice.grid_size(level)
        op = {}
        # the operator surrogate replaces the assembled residual only for the surrogate smoother
        # (reference multigrid.py:418: use_surrogate_a = a_mode == 'surrogate' and kind == 'surrogate_ilu')
        if config.a_mode == "surrogate" and config.kind == "surrogate_ilu":
            op["acoefs"] = fitting.fit_surrogate_operator(source, level, config.a_degrees, config.sample_level)
        elif source.sepk is not None:
            op["sepk"] = source.sepk          # rows evaluated on the fly: nothing per point uploaded
        elif source.constant:
            op["arow"] = np.atleast_1d(source.data)
        else:
            op["arows"] = source.data
        if config.kind == "ilu":
            self.factorization = (fitting.factorize_tet_device(source, level, keep_on_device=True)
                                  if factorize == "device" else fitting.factorize_tet(source, level))
            self.precond = CellILU(self.factorization)
            self.plan = DevicePlan(level, np.zeros((7, 1, 1, 1)), np.zeros(1), "v2",
                                   factors=self.factorization.rows, fast=fast, simple=simple, **op)
            self._stored = True
        else:
            self.precond = build_surrogate_ilu(source, level, config.degrees, config.variant,
                                               config.sample_level, fast=fast, factorize=factorize)
            self.plan = self.precond.plan(simple=simple, **op)
            self._stored = False

    @classmethod
    def setup(cls, source, level: int | None = None, degrees=(3, 3, 3), variant: str = "v1",
              sample_level=None, *, coeff: CoefficientField | None = None, kind: str = "surrogate_ilu",
              a_mode: str = "assembled", a_degrees=(3, 3, 3), fast: bool = False, simple: bool = False,
              factorize: str = "host"):
        """``source`` is a StencilSource, or macro-tet vertices (4, 3) plus ``coeff``.  ``factorize``:
        where the ILU(0) factorization sweep of the setup runs ("host" or "device", same rows bitwise)."""
        if not isinstance(source, StencilSource):
            if level is None:
                raise ValueError("level is required when passing vertices")
            source = stencil_source(source, level, coeff or CoefficientField.constant(1.0))
        level = source.level if level is None else level
        cfg = SmootherConfig(kind, tuple(degrees), variant, sample_level, a_mode, tuple(a_degrees))
        return cls(source, level, cfg, fast=fast, simple=simple, factorize=factorize)

    @property
    def degrees(self):
        return getattr(self.precond, "degrees", None)

    def solve_into(self, w) -> None:
        self.precond.solve_into(w) if not isinstance(w, torch.Tensor) else (
            self.plan.stored_solve_into(w) if self._stored else self.plan.solve_into(w))

    def residual(self, u, f, w=None, norms: bool = False):
        return self.plan.residual(u, f, w, norms)

    def apply(self, u, f, sweeps: int = 1, *, residual_norms: bool = False, check_finite: bool = False):
        """In place on u (CUDA fp64 [grid] or [ntets, grid] sharing this operator).
        Returns ||f - A u||^2 before each sweep ([sweeps, ntets]) if ``residual_norms``.
        ``check_finite`` (implies the norms; synchronises the stream): raise FloatingPointError when a
        residual norm is NaN or infinite -- a diverged or corrupted iterate is reported, not propagated."""
        residual_norms = residual_norms or check_finite
        host = isinstance(u, np.ndarray)
        if host:
            ut = torch.as_tensor(np.ascontiguousarray(u), device="cuda")
            ft = torch.as_tensor(np.ascontiguousarray(f), device="cuda")
        else:
            ut, ft = u, f
        rn = self.plan.sweep(ut, ft, sweeps, norms=residual_norms, stored=self._stored)
        if check_finite and not bool(torch.isfinite(rn).all()):
            bad = torch.nonzero(~torch.isfinite(rn))[0].tolist()
            raise FloatingPointError(f"non-finite residual norm before sweep {bad[0]} (tet {bad[1]})")
        if host:
            u[...] = ut.cpu().numpy()
            rn = None if rn is None else rn.cpu().numpy()
        return rn

    def apply_many(self, us, fs, sweeps: int = 1, *, residual_norms: bool = False, check_finite: bool = False):
        return self.apply(us, fs, sweeps, residual_norms=residual_norms, check_finite=check_finite)

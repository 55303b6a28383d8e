"""Multigrid V-cycle around the GPU smoother on one all-Dirichlet macro-tetrahedron.

Mirror of the reference ``Hierarchy`` (multigrid.py:306-513) for ``mesh = single_tet_mesh`` -- the
caller of the hot path: identity DoF numbering, free = interior, no interface primitives
(multigrid.py:100-108), so one smoother application is the cell stage alone.  Everything of the cycle
runs on the device: the smoothing sweeps (``tilu_sweep``), the residual (``tilu_residual``), the
restriction / prolongation (``tilu_mg_restrict`` / ``tilu_mg_prolong_add``, the matrix-free form of
``build_prolongation``, multigrid.py:241-277) and the coarsest-level solve (a dense inverse applied by
``tilu_dense_mv`` in place of the reference's PCG to 1e-12, multigrid.py:445-457).  Vectors are CUDA
float64 tensors in the reference layout (full-lattice rank order, zero outside the interior).

Residuals use the stencil rows (``stencil_apply`` form) where the reference multiplies by the assembled
CSR matrix; the two differ by rounding only (<= 8.2e-15 relative).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib, lattice
from .smoother import SmootherConfig, SurrogateILUSmoother
from .stencil import CoefficientField, StencilSource, stencil_source


def interior_matrix(source: StencilSource) -> np.ndarray:
    """Dense interior block of the level operator from its stencil rows (coarsest level only)."""
    level = source.level
    inner = lattice.lattice_coords(level, "interior")
    ranks = lattice.lattice_rank(inner, level)
    pos = {int(r): i for i, r in enumerate(ranks)}
    m = len(inner)
    A = np.zeros((m, m))
    for i, p in enumerate(inner):
        row = source.data if source.constant else source.data[ranks[i]]
        for d in range(15):
            q = p + lattice.OFFSETS[d]
            if lattice.is_interior(q[None], level)[0]:
                A[i, pos[int(lattice.lattice_rank(q[None], level)[0])]] = row[d]
    return A


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


class Hierarchy:
    """Levels ``lmin`` (direct solve) .. ``lmax`` on one macro-tet; same knobs as the reference's
    ``Hierarchy(mesh, lmin, lmax, coeff, smoother=SmootherConfig, nu_pre, nu_post)``."""

    def __init__(self, tet, lmin: int = 2, lmax: int = 6, coeff: CoefficientField | None = None,
                 smoother: SmootherConfig | None = None, nu_pre: int = 3, nu_post: int = 3,
                 fast: bool = False, factorize: str = "host", device="cuda", max_coarse_dofs: int = 4096):
        if not 2 <= lmin <= lmax:
            raise ValueError("need 2 <= lmin <= lmax")
        self.tet = np.asarray(getattr(tet, "vertices", tet), dtype=np.float64)
        self.levels = list(range(lmin, lmax + 1))
        self.coeff = coeff if coeff is not None else CoefficientField.constant(1.0)
        self.smoother_config = smoother if smoother is not None else SmootherConfig()
        self.nu_pre, self.nu_post = int(nu_pre), int(nu_post)
        self.device = torch.device(device)
        self.sources = [stencil_source(self.tet, l, self.coeff) for l in self.levels]
        if lattice.interior_size(lmin) > max_coarse_dofs:
            raise ValueError(f"coarsest level {lmin} has {lattice.interior_size(lmin)} DoF: too many for the dense solve")
        # coarsest level: dense inverse of the interior block (the reference runs PCG to 1e-12 |b|)
        A0 = interior_matrix(self.sources[0])
        self._coarse_inv = torch.as_tensor(np.linalg.inv(A0) if len(A0) else A0, device=self.device)
        self._coarse_idx = torch.as_tensor(
            lattice.lattice_rank(lattice.lattice_coords(lmin, "interior"), lmin), device=self.device)
        # smoothers of the levels above the coarsest (built eagerly: setup belongs to the constructor)
        self.smoothers = [None] + [
            SurrogateILUSmoother(src, l, self.smoother_config, fast=fast, factorize=factorize)
            for src, l in zip(self.sources[1:], self.levels[1:])]
        # residual / correction scratch per level
        self._r = [torch.zeros(lattice.grid_size(l), dtype=torch.float64, device=self.device) for l in self.levels]
        self._e = [torch.zeros(lattice.grid_size(l), dtype=torch.float64, device=self.device) for l in self.levels]
        self._rc = [torch.zeros(lattice.grid_size(l), dtype=torch.float64, device=self.device) for l in self.levels]
        self._free = [torch.as_tensor(lattice.interior_mask(l), device=self.device) for l in self.levels]

    @property
    def top(self) -> int:
        return len(self.levels) - 1

    def zero(self, li: int) -> torch.Tensor:
        return torch.zeros(lattice.grid_size(self.levels[li]), dtype=torch.float64, device=self.device)

    def _check(self, li: int, *vs) -> None:
        g = lattice.grid_size(self.levels[li])
        for v in vs:
            if not (isinstance(v, torch.Tensor) and v.is_cuda and v.dtype == torch.float64 and v.is_contiguous()
                    and v.numel() == g):
                raise ValueError(f"level {self.levels[li]} vectors must be contiguous CUDA float64 tensors of {g} entries")

    # -- transfers (multigrid.py:377-388) ---------------------------------------------------------

    def restrict(self, li: int, r_fine: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """P^T r from level index li to li - 1 (r zero outside the interior)."""
        if li == 0:
            raise ValueError("already on the coarsest level")
        self._check(li, r_fine)
        out = self.zero(li - 1) if out is None else out
        _lib.check(_lib.lib().tilu_mg_restrict(self.levels[li - 1], r_fine.data_ptr(), out.data_ptr(), _stream()))
        return out

    def prolongate_add(self, li: int, e_coarse: torch.Tensor, u_fine: torch.Tensor) -> None:
        """u_fine += P e_coarse (level index li - 1 to li), interior points only."""
        if li == 0:
            raise ValueError("no level below the coarsest")
        self._check(li, u_fine)
        self._check(li - 1, e_coarse)
        _lib.check(_lib.lib().tilu_mg_prolong_add(self.levels[li - 1], e_coarse.data_ptr(), u_fine.data_ptr(), _stream()))

    # -- smoother, coarse solve, cycle (multigrid.py:431-485) ---------------------------------------

    def smooth(self, li: int, u: torch.Tensor, f: torch.Tensor, steps: int = 1) -> None:
        self.smoothers[li].apply(u, f, steps)

    def residual(self, li: int, u: torch.Tensor, f: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        if li == 0:
            raise ValueError("the coarsest level is solved directly")
        self.smoothers[li].residual(u, f, out)
        return out

    def coarse_solve(self, u: torch.Tensor, f: torch.Tensor) -> None:
        m = self._coarse_idx.numel()
        if m == 0:
            return
        b = f.index_select(0, self._coarse_idx).contiguous()
        x = torch.empty_like(b)
        _lib.check(_lib.lib().tilu_dense_mv(m, self._coarse_inv.data_ptr(), b.data_ptr(), x.data_ptr(), _stream()))
        u.index_copy_(0, self._coarse_idx, x)

    def v_cycle(self, li: int, u: torch.Tensor, f: torch.Tensor) -> None:
        """Standard V-cycle, in place on u (multigrid.py:459-485)."""
        self._check(li, u, f)
        if li == 0:
            self.coarse_solve(u, f)
            return
        if self.nu_pre:
            self.smooth(li, u, f, self.nu_pre)
        r = self.residual(li, u, f, self._r[li])
        rc = self.restrict(li, r, self._rc[li - 1])
        ec = self._e[li - 1]
        ec.zero_()
        self.v_cycle(li - 1, ec, rc)
        self.prolongate_add(li, ec, u)
        if self.nu_post:
            self.smooth(li, u, f, self.nu_post)

    def solve(self, f: torch.Tensor, tol: float = 1e-10, max_cycles: int = 100, u0: torch.Tensor | None = None):
        """V-cycle iteration until the relative residual drops below tol (multigrid.py:487-503)."""
        li = self.top
        if li == 0:
            u = self.zero(0)
            self.coarse_solve(u, f)
            return u, 1
        u = self.zero(li) if u0 is None else u0.clone()
        b = torch.where(self._free[li], f, torch.zeros_like(f))
        nb = float(torch.linalg.norm(b))
        if nb == 0.0:
            return u, 0
        r = self.zero(li)
        for k in range(1, max_cycles + 1):
            self.v_cycle(li, u, b)
            if float(torch.linalg.norm(self.residual(li, u, b, r))) <= tol * nb:
                return u, k
        return u, max_cycles

    def convergence_factor(self, steps: int = 20, seed: int = 42) -> float:
        """Asymptotic error-reduction factor of the V-cycle: normalised power iteration on the error
        propagator, f = 0 (multigrid.py:505-523; same seed convention: the normal draw covers every
        lattice point, boundary entries are then zeroed)."""
        li = self.top
        g = lattice.grid_size(self.levels[li])
        e0 = np.random.default_rng(seed).standard_normal(g)
        e0[~lattice.interior_mask(self.levels[li])] = 0.0
        e0 /= np.linalg.norm(e0)
        e = torch.as_tensor(e0, device=self.device)
        f = self.zero(li)
        rho = 0.0
        for _ in range(steps):
            self.v_cycle(li, e, f)
            rho = float(torch.linalg.norm(e))
            if not np.isfinite(rho) or rho == 0.0:
                raise RuntimeError("power iteration collapsed")
            e /= rho
        return rho


class InnerSolveError(RuntimeError):
    """The inner multigrid of a Schur interior solve stalled (reference schur.py:27-28)."""


def schur_inner_solve(hier: Hierarchy, rhs: torch.Tensor, tol: float = 1e-8, max_cycles: int = 50) -> torch.Tensor:
    """Interior solve A_tt^{-1} rhs of one macro-tet by V-cycles with the configured smoother -- the
    'multigrid' branch of the reference's SchurComplement._inner_solve (schur.py:80-100): rhs holds the
    interior DoF in lattice-rank order; returns the interior solution (CUDA tensors).  Raises
    InnerSolveError when the residual stays above 10 tol |f| (schur.py:96-99)."""
    lvl = hier.levels[hier.top]
    if rhs.dim() != 1 or rhs.numel() != lattice.interior_size(lvl):
        raise ValueError(f"rhs must hold the {lattice.interior_size(lvl)} interior DoF of level {lvl}")
    idx = torch.as_tensor(lattice.lattice_rank(lattice.lattice_coords(lvl, "interior"), lvl), device=hier.device)
    f = hier.zero(hier.top)
    f.index_copy_(0, idx, rhs.to(hier.device, torch.float64))
    u, _ = hier.solve(f, tol=tol, max_cycles=max_cycles)
    r = hier.residual(hier.top, u, f, hier.zero(hier.top)) if hier.top > 0 else torch.zeros_like(f)
    resid, nf = float(torch.linalg.norm(r)), float(torch.linalg.norm(f))
    if resid > 10 * tol * nf:
        raise InnerSolveError(f"inner multigrid stalled (residual {resid:.2e})")
    return u.index_select(0, idx)

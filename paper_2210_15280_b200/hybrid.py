"""Hybrid multi-tet smoother on the GPU: the reference's primitive-sequence smoother
``Hierarchy.smooth`` (multigrid.py:431-442) for macro-meshes whose tets share vertices, edges and faces.

One application = interface stages (vertex, edge, face: CSR lower substitution on the residual of each
primitive block, ``_interface_stage`` multigrid.py:400-412), the cell stage (every macro-tet interior:
the ILU(0) / surrogate sweep of this library, ``_cell_stage`` multigrid.py:414-429) and, for the
symmetric smoother, the interface stages in reverse with the transposed (upper) substitution.

The mesh bookkeeping stays with the caller (the reference's ``LevelSpace``: global numbering, assembled
matrix, primitive DoF lists); this class takes those arrays -- ``A`` (scipy CSR), ``prim_dofs``
({"vertex" | "edge" | "face": [global ids per primitive]}), ``cell_dof`` ([ntets][grid] global id of every
local lattice point) -- and runs every stage on the device.  INTEGRATION.md shows the binding inside the
reference ``Hierarchy``.  Interface stages are bitwise the reference's; the cell stage computes its
residual in stencil form (the reference multiplies by the CSR matrix: same value up to rounding).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib, lattice
from .partition import group_by_operator
from .smoother import SmootherConfig, SurrogateILUSmoother
from .stencil import CoefficientField, stencil_source


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _check_vec(name: str, v, n: int, device) -> None:
    """The kernels index the vectors with the mesh's global ids: wrong sizes / dtypes / devices must fail here,
    not read past an allocation."""
    if not (isinstance(v, torch.Tensor) and v.is_cuda and v.dtype == torch.float64 and v.is_contiguous()
            and v.dim() == 1 and v.numel() == n):
        raise ValueError(f"{name} must be a contiguous CUDA float64 vector of {n} entries")
    if v.device != torch.device(device) and torch.device(device).index is not None:
        raise ValueError(f"{name} is on {v.device}, the smoother on {device}")


def _schedule(blocks, upper: bool):
    """Level schedule of every block: (loff [nb+1], lptr [nlev+1], perm [nrows])."""
    L = _lib.lib()
    loff, lptr, perm = [0], [0], []
    for blk in blocks:
        m = blk.shape[0]
        indptr = np.ascontiguousarray(blk.indptr, dtype=np.int64)
        indices = np.ascontiguousarray(blk.indices, dtype=np.int32)
        level = np.zeros(max(m, 1), dtype=np.int32)
        nl = L.tilu_csr_levels(m, indptr.ctypes.data, indices.ctypes.data, int(upper), level.ctypes.data)
        if nl < 0:
            raise ValueError("bad CSR block")
        order = np.argsort(level[:m], kind="stable").astype(np.int32)
        counts = np.bincount(level[:m], minlength=nl)
        for c in counts:
            lptr.append(lptr[-1] + int(c))
        perm.append(order)
        loff.append(loff[-1] + nl)
    perm = np.concatenate(perm) if perm else np.empty(0, np.int32)
    return np.array(loff, np.int64), np.array(lptr, np.int64), perm.astype(np.int32)


class InterfaceStage:
    """All primitive blocks of one kind at one level (reference ``Hierarchy._blocks`` +
    ``_interface_stage``, multigrid.py:362-371, 400-412)."""

    def __init__(self, A, ids_list, device="cuda"):
        dev = torch.device(device)
        self.nblocks = len(ids_list)
        if self.nblocks == 0:
            return
        A = A.tocsr()
        ids = np.concatenate([np.asarray(i, dtype=np.int64) for i in ids_list])
        rows = A[ids].tocsr()
        rows.sort_indices()
        blocks = []
        for i in ids_list:
            b = A[np.ix_(i, i)].tocsr()
            b.sort_indices()
            blocks.append(b)
        roff = np.cumsum([0] + [b.shape[0] for b in blocks]).astype(np.int64)
        nnz_off = np.cumsum([0] + [b.nnz for b in blocks]).astype(np.int64)
        indptr = np.concatenate([b.indptr[:-1].astype(np.int64) + nnz_off[k] for k, b in enumerate(blocks)]
                                + [nnz_off[-1:]])
        t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a, dtype=dt), device=dev)  # noqa: E731
        self.n = len(ids)
        self.ids = t(ids, np.int64)
        self.r_indptr, self.r_indices, self.r_data = t(rows.indptr, np.int64), t(rows.indices, np.int64), t(rows.data, np.float64)
        self.roff, self.indptr = t(roff, np.int64), t(indptr, np.int64)
        self.indices = t(np.concatenate([b.indices for b in blocks]), np.int32)
        self.data = t(np.concatenate([b.data for b in blocks]), np.float64)
        self.sched = [tuple(t(a, a.dtype) for a in _schedule(blocks, upper)) for upper in (False, True)]
        self.r = torch.empty(self.n, dtype=torch.float64, device=dev)
        self.z = torch.empty(self.n, dtype=torch.float64, device=dev)

    def apply(self, u: torch.Tensor, f: torch.Tensor, transposed: bool = False) -> None:
        """u[ids] += T^{-1} (f - A u)[ids] per block, T the lower (transposed: upper) triangle incl. diagonal."""
        if self.nblocks == 0:
            return
        L = _lib.lib()
        _lib.check(L.tilu_csr_residual_rows(self.n, self.r_indptr.data_ptr(), self.r_indices.data_ptr(),
                                            self.r_data.data_ptr(), self.ids.data_ptr(), u.data_ptr(), f.data_ptr(),
                                            self.r.data_ptr(), _stream()))
        loff, lptr, perm = self.sched[int(transposed)]
        _lib.check(L.tilu_csr_tri_solve_blocks(self.nblocks, self.roff.data_ptr(), self.indptr.data_ptr(),
                                               self.indices.data_ptr(), self.data.data_ptr(), loff.data_ptr(),
                                               lptr.data_ptr(), perm.data_ptr(), int(transposed), self.r.data_ptr(),
                                               self.z.data_ptr(), self.ids.data_ptr(), u.data_ptr(), _stream()))


class HybridSmoother:
    """``smooth(u, f)`` = one application of the reference's primitive-sequence smoother on a macro-mesh."""

    def __init__(self, A, prim_dofs: dict, cell_dof, tets, level: int, coeff: CoefficientField | None = None,
                 config: SmootherConfig | None = None, symmetric: bool = True, fast: bool = False,
                 factorize: str = "host", device="cuda"):
        self.level = int(level)
        self.symmetric = bool(symmetric)
        self.device = torch.device(device)
        self.ndof = int(A.shape[0])
        if A.shape[0] != A.shape[1]:
            raise ValueError("A must be square")
        self.config = config if config is not None else SmootherConfig()
        coeff = coeff if coeff is not None else CoefficientField.constant(1.0)
        self.stages = {k: InterfaceStage(A, [np.asarray(i) for i in prim_dofs.get(k, [])], device)
                       for k in ("vertex", "edge", "face")}
        cell_dof = np.asarray(cell_dof, dtype=np.int64)
        grid = lattice.grid_size(level)
        if cell_dof.ndim != 2 or cell_dof.shape[1] != grid:
            raise ValueError(f"cell_dof must be [ntets, {grid}]")
        if cell_dof.size and (cell_dof.min() < 0 or cell_dof.max() >= self.ndof):
            raise ValueError("cell_dof holds ids outside the matrix")
        for k in ("vertex", "edge", "face"):
            for ids in prim_dofs.get(k, []):
                ids = np.asarray(ids)
                if ids.size and (ids.min() < 0 or ids.max() >= self.ndof):
                    raise ValueError(f"{k} primitive holds ids outside the matrix")
        self.ntets = cell_dof.shape[0]
        sources = [stencil_source(np.asarray(t, dtype=np.float64), level, coeff) for t in tets]
        if len(sources) != self.ntets:
            raise ValueError("one macro-tet per row of cell_dof")
        # tets with identical operator rows share one plan and run as one batch
        self.groups = group_by_operator([s.data for s in sources])
        self.smoothers = [SurrogateILUSmoother(sources[g[0]], level, self.config, fast=fast, factorize=factorize)
                          for g in self.groups]
        imask = lattice.interior_mask(level)
        self._gather = [torch.as_tensor(cell_dof[g], device=self.device) for g in self.groups]            # [T, grid]
        self._interior = [torch.as_tensor(cell_dof[g][:, imask], device=self.device) for g in self.groups]  # [T, N]
        self._imask = torch.as_tensor(imask, device=self.device)

    def interface_stage(self, u, f, kind: str, transposed: bool = False) -> None:
        _check_vec("u", u, self.ndof, self.device)
        _check_vec("f", f, self.ndof, self.device)
        self.stages[kind].apply(u, f, transposed)

    def cell_stage(self, u: torch.Tensor, f: torch.Tensor) -> None:
        """Every macro-tet interior: u_t += M_t^{-1} (f - A u)_t with the tet's boundary values taken from
        the global vector (multigrid.py:414-429).  All tets read the same u (block Jacobi across cells)."""
        _check_vec("u", u, self.ndof, self.device)
        _check_vec("f", f, self.ndof, self.device)
        locs = []
        for sm, gidx in zip(self.smoothers, self._gather):
            ul = u[gidx].contiguous()
            fl = f[gidx].contiguous()
            sm.apply(ul, fl, 1)
            locs.append(ul)
        for ul, iidx in zip(locs, self._interior):
            u[iidx.reshape(-1)] = ul[:, self._imask].reshape(-1)

    def smooth(self, u: torch.Tensor, f: torch.Tensor) -> None:
        for kind in ("vertex", "edge", "face"):
            self.interface_stage(u, f, kind, False)
        self.cell_stage(u, f)
        if self.symmetric:
            for kind in ("face", "edge", "vertex"):
                self.interface_stage(u, f, kind, True)


class _DevCSR:
    """A scipy CSR matrix on the device (int64 indices, sorted) for tilu_csr_matvec / tilu_csr_residual_rows."""

    def __init__(self, M, device):
        M = M.tocsr()
        M.sort_indices()
        self.shape = M.shape
        t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a, dtype=dt), device=device)  # noqa: E731
        self.indptr, self.indices, self.data = t(M.indptr, np.int64), t(M.indices, np.int64), t(M.data, np.float64)

    def matvec(self, x: torch.Tensor, y: torch.Tensor, accumulate: bool = False) -> torch.Tensor:
        _lib.check(_lib.lib().tilu_csr_matvec(self.shape[0], self.indptr.data_ptr(), self.indices.data_ptr(),
                                              self.data.data_ptr(), x.data_ptr(), y.data_ptr(), int(accumulate), _stream()))
        return y


class HybridHierarchy:
    """Multigrid V-cycle on a macro-mesh whose tets share primitives: the reference ``Hierarchy`` (multigrid.py:
    306-523) with every operation of the cycle on the device -- the hybrid smoother (interface stages + cell
    stage), the residual with the assembled matrix, the transfers P e / P^T r with the caller's prolongation
    matrices in scipy's accumulation order, and a dense solve on the coarsest level (the reference: PCG to
    1e-12).  The mesh bookkeeping is the caller's (per level li: ``A[li]`` scipy CSR, ``P[li]`` from level li to
    li + 1, ``prim_dofs[li]``, ``cell_dof[li]``, ``free[li]``), exactly the arrays the reference ``Hierarchy``
    holds (``H.A``, ``H.P``, ``H.spaces[li].prim_dofs / cell_dof / free``)."""

    def __init__(self, levels, A, P, prim_dofs, cell_dof, free, tets, coeff: CoefficientField | None = None,
                 smoother: SmootherConfig | None = None, nu_pre: int = 3, nu_post: int = 3, symmetric: bool = True,
                 fast: bool = False, factorize: str = "host", device="cuda"):
        self.levels = [int(l) for l in levels]
        nl = len(self.levels)
        if not (len(A) == nl and len(P) == nl - 1 and len(prim_dofs) == nl and len(cell_dof) == nl and len(free) == nl):
            raise ValueError("one A / prim_dofs / cell_dof / free per level and one P per level pair")
        self.device = torch.device(device)
        self.nu_pre, self.nu_post = int(nu_pre), int(nu_post)
        self.ndof = [int(a.shape[0]) for a in A]
        self.free = [torch.as_tensor(np.asarray(m, dtype=bool), device=self.device) for m in free]
        self.smoothers = [None] + [HybridSmoother(A[li], prim_dofs[li], cell_dof[li], tets, self.levels[li], coeff,
                                                  smoother, symmetric=symmetric, fast=fast, factorize=factorize,
                                                  device=device) for li in range(1, nl)]
        self.A = [None] + [_DevCSR(A[li], self.device) for li in range(1, nl)]
        self._rows = [None] + [torch.arange(self.ndof[li], dtype=torch.int64, device=self.device) for li in range(1, nl)]
        self.P = [_DevCSR(p, self.device) for p in P]
        self.PT = [_DevCSR(p.T, self.device) for p in P]
        f0 = np.nonzero(np.asarray(free[0], dtype=bool))[0]
        A0 = A[0].tocsr()[np.ix_(f0, f0)].toarray()
        self._coarse_idx = torch.as_tensor(f0, device=self.device)
        self._coarse_inv = torch.as_tensor(np.linalg.inv(A0) if len(f0) else A0, device=self.device)
        z = lambda li: torch.zeros(self.ndof[li], dtype=torch.float64, device=self.device)  # noqa: E731
        self._r = [z(li) for li in range(nl)]
        self._rc = [z(li) for li in range(nl)]
        self._e = [z(li) for li in range(nl)]

    @property
    def top(self) -> int:
        return len(self.levels) - 1

    def zero(self, li: int) -> torch.Tensor:
        return torch.zeros(self.ndof[li], dtype=torch.float64, device=self.device)

    def smooth(self, li: int, u: torch.Tensor, f: torch.Tensor) -> None:
        self.smoothers[li].smooth(u, f)

    def residual(self, li: int, u: torch.Tensor, f: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        """out = f - A u on free DoF, 0 elsewhere (multigrid.py:474-475)."""
        a = self.A[li]
        _lib.check(_lib.lib().tilu_csr_residual_rows(self.ndof[li], a.indptr.data_ptr(), a.indices.data_ptr(),
                                                     a.data.data_ptr(), self._rows[li].data_ptr(), u.data_ptr(),
                                                     f.data_ptr(), out.data_ptr(), _stream()))
        out.masked_fill_(~self.free[li], 0.0)
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
        """In place on u (multigrid.py:459-485)."""
        _check_vec("u", u, self.ndof[li], self.device)
        _check_vec("f", f, self.ndof[li], self.device)
        if li == 0:
            self.coarse_solve(u, f)
            return
        for _ in range(self.nu_pre):
            self.smooth(li, u, f)
        r = self.residual(li, u, f, self._r[li])
        rc = self.PT[li - 1].matvec(r, self._rc[li - 1])
        rc.masked_fill_(~self.free[li - 1], 0.0)
        ec = self._e[li - 1]
        ec.zero_()
        self.v_cycle(li - 1, ec, rc)
        self.P[li - 1].matvec(ec, u, accumulate=True)
        u.masked_fill_(~self.free[li], 0.0)
        for _ in range(self.nu_post):
            self.smooth(li, u, f)

    def convergence_factor(self, steps: int = 20, seed: int = 42) -> float:
        """Normalised power iteration on the error propagator, f = 0 (multigrid.py:505-523)."""
        li = self.top
        e0 = np.random.default_rng(seed).standard_normal(self.ndof[li])
        e0[~self.free[li].cpu().numpy()] = 0.0
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

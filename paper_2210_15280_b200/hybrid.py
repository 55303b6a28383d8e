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
        self.config = config if config is not None else SmootherConfig()
        coeff = coeff if coeff is not None else CoefficientField.constant(1.0)
        self.stages = {k: InterfaceStage(A, [np.asarray(i) for i in prim_dofs.get(k, [])], device)
                       for k in ("vertex", "edge", "face")}
        cell_dof = np.asarray(cell_dof, dtype=np.int64)
        grid = lattice.grid_size(level)
        if cell_dof.ndim != 2 or cell_dof.shape[1] != grid:
            raise ValueError(f"cell_dof must be [ntets, {grid}]")
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
        self.stages[kind].apply(u, f, transposed)

    def cell_stage(self, u: torch.Tensor, f: torch.Tensor) -> None:
        """Every macro-tet interior: u_t += M_t^{-1} (f - A u)_t with the tet's boundary values taken from
        the global vector (multigrid.py:414-429).  All tets read the same u (block Jacobi across cells)."""
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

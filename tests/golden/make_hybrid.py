"""Golden fixtures for the hybrid smoother's interface stages.

Runs the UNMODIFIED reference (``/root/reference/pkg/src/tetilu``, build container only) on its
``cube_mesh`` (12 macro-tets, Dirichlet top / bottom, natural sides: shared vertices, edges and faces):
the global numbering and matrix of ``LevelSpace`` / ``Hierarchy``, every ``_interface_stage`` alone
(lower and transposed, multigrid.py:400-412 -> _kernels.csr_lower/upper_solve, _kernels.py:490-519) and
full ``smooth`` steps (multigrid.py:431-442).  Writes ``tests/golden/hybrid_L*.npz``.

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_hybrid.py
"""

from __future__ import annotations

import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import numpy as np  # noqa: E402

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from tetilu import geometry  # noqa: E402
from tetilu.multigrid import Hierarchy, SmootherConfig  # noqa: E402


def case(level, cfg, inputs_from=None):
    mesh = geometry.cube_mesh()
    H = Hierarchy(mesh, lmin=level, lmax=level, smoother=cfg)
    li = H.top
    sp = H.spaces[li]
    A = H.A[li].tocsr()
    A.sort_indices()
    rng = np.random.default_rng(7)
    u0 = np.where(sp.free, rng.uniform(-1, 1, sp.ndof), 0.0)
    f = np.where(sp.free, rng.standard_normal(sp.ndof), 0.0)
    out = dict(level=level, ndof=sp.ndof, indptr=A.indptr.astype(np.int64), indices=A.indices.astype(np.int64),
               data=A.data, free=sp.free, u0=u0, f=f,
               cell_dof=np.stack(sp.cell_dof), tets=np.stack([mesh.cell_tet(ci).vertices for ci in range(mesh.num_cells)]),
               kind=cfg.kind, degrees=np.array(cfg.degrees), variant=cfg.variant, symmetric=cfg.symmetric)
    for kind in ("vertex", "edge", "face"):
        ids = sp.prim_dofs[kind]
        out[f"{kind}_ids"] = np.concatenate(ids) if ids else np.empty(0, np.int64)
        out[f"{kind}_off"] = np.cumsum([0] + [len(i) for i in ids]).astype(np.int64)
        for transposed in (False, True):
            u = u0.copy()
            H._interface_stage(li, u, f, kind, transposed)
            out[f"stage_{kind}_{int(transposed)}"] = u
    u = u0.copy()
    steps = []
    for _ in range(2):
        H.smooth(li, u, f)
        steps.append(u.copy())
    out["u_smooth"] = np.stack(steps)
    u = u0.copy()
    H._cell_stage(li, u, f)
    out["u_cell_stage"] = u
    if inputs_from:   # same mesh / vectors as another case: keep only what differs
        out = {k: out[k] for k in ("level", "kind", "degrees", "variant", "symmetric", "u_smooth", "u_cell_stage")}
        out["inputs_from"] = inputs_from
    np.savez_compressed(os.path.join(OUT, f"hybrid_L{level}_{cfg.kind}.npz"), **out)
    print(level, cfg.kind, sp.ndof, {k: len(sp.prim_dofs[k]) for k in ("vertex", "edge", "face")},
          float(np.abs(steps[-1]).max()))


if __name__ == "__main__":
    case(3, SmootherConfig(kind="surrogate_ilu", degrees=(2, 2, 2), variant="v1"))
    case(4, SmootherConfig(kind="surrogate_ilu", degrees=(3, 3, 3), variant="v1"))
    case(4, SmootherConfig(kind="ilu"), inputs_from="hybrid_L4_surrogate_ilu")

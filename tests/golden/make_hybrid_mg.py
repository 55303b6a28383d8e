"""Golden fixture for the multigrid V-cycle on a macro-mesh with shared primitives (SURVEY 8(f)2 + 8(f)4).

Runs the UNMODIFIED reference (``/root/reference/pkg/src/tetilu``, build container only): ``Hierarchy`` on its
``cube_mesh`` (12 macro-tets), levels 2..4, the hybrid primitive-sequence smoother inside the V-cycle.  Stores
the reference's bookkeeping the device hierarchy is bound to (per level: assembled matrix, primitive DoF lists,
cell numbering, free mask; prolongations) and its results (iterates of three V-cycles, convergence factor).
Level-4 arrays are shared with tests/golden/hybrid_L4_surrogate_ilu.npz (same mesh and coefficient).

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_hybrid_mg.py
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

if __name__ == "__main__":
    mesh = geometry.cube_mesh()
    cfg = SmootherConfig(kind="surrogate_ilu", degrees=(3, 3, 3), variant="v1")
    H = Hierarchy(mesh, lmin=2, lmax=4, smoother=cfg, nu_pre=2, nu_post=2)
    out = dict(levels=np.array(H.levels), nu=2, kind=cfg.kind, degrees=np.array(cfg.degrees), variant=cfg.variant,
               symmetric=cfg.symmetric, top_from="hybrid_L4_surrogate_ilu")
    for li, sp in enumerate(H.spaces):
        if li < H.top:       # the top level's arrays live in hybrid_L4_surrogate_ilu.npz
            A = H.A[li].tocsr()
            A.sort_indices()
            out[f"A{li}_indptr"], out[f"A{li}_indices"], out[f"A{li}_data"] = (
                A.indptr.astype(np.int64), A.indices.astype(np.int64), A.data)
            out[f"free{li}"] = sp.free
            out[f"cell_dof{li}"] = np.stack(sp.cell_dof)
            for kind in ("vertex", "edge", "face"):
                ids = sp.prim_dofs[kind]
                out[f"{kind}{li}_ids"] = np.concatenate(ids) if ids else np.empty(0, np.int64)
                out[f"{kind}{li}_off"] = np.cumsum([0] + [len(i) for i in ids]).astype(np.int64)
            P = H.P[li].tocsr()
            P.sort_indices()
            out[f"P{li}_indptr"], out[f"P{li}_indices"], out[f"P{li}_data"] = (
                P.indptr.astype(np.int64), P.indices.astype(np.int64), P.data)
            out[f"P{li}_shape"] = np.array(P.shape)
    sp = H.spaces[H.top]
    rng = np.random.default_rng(21)
    f = np.where(sp.free, rng.standard_normal(sp.ndof), 0.0)
    u = np.zeros(sp.ndof)
    us = []
    for _ in range(3):
        H.v_cycle(H.top, u, f)
        us.append(u.copy())
    out["f"] = f
    out["u_cycles"] = np.stack(us)
    out["rho"] = H.convergence_factor(steps=8, seed=42)
    out["rho_steps"] = 8
    np.savez_compressed(os.path.join(OUT, "hybrid_mg_L4.npz"), **out)
    print("rho", out["rho"], [float(np.abs(v).max()) for v in us], os.path.getsize(os.path.join(OUT, "hybrid_mg_L4.npz")))

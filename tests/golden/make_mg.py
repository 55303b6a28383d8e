"""Golden fixtures for the multigrid cycle around the smoother and the transfers.

Runs the UNMODIFIED reference (``/root/reference/pkg/src/tetilu``, importable in the build container
only): ``Hierarchy`` on ``single_tet_mesh`` (all faces Dirichlet), its prolongation matrices, V-cycles
and ``convergence_factor``.  Writes ``tests/golden/mg_*.npz``; the GPU box never reads /root/reference.

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_mg.py
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
from tetilu.assembly import CoefficientField  # noqa: E402
from tetilu.multigrid import Hierarchy, SmootherConfig  # noqa: E402

UNIT = geometry.trirect_tet(1.0)
DISTORTED = np.array([(0, 0, 0), (1, 0.1, 0), (0.2, 1, 0), (0.1, 0.3, 0.8)], dtype=float)


def diag_tensor(d):
    d = np.asarray(d, dtype=float)
    return CoefficientField.tensor(lambda pts: np.broadcast_to(np.diag(d), (len(np.atleast_2d(pts)), 3, 3)))


def case(name, tet, coeff, lmin, lmax, cfg, nu, cycles=3, steps=8):
    mesh = geometry.single_tet_mesh(tet)
    H = Hierarchy(mesh, lmin=lmin, lmax=lmax, coeff=coeff, smoother=cfg, nu_pre=nu, nu_post=nu)
    top = H.top
    sp = H.spaces[top]
    rng = np.random.default_rng(11)
    f = np.where(sp.free, rng.standard_normal(sp.ndof), 0.0)
    u = np.zeros(sp.ndof)
    us = []
    for _ in range(cycles):
        H.v_cycle(top, u, f)
        us.append(u.copy())
    rho = H.convergence_factor(steps=steps, seed=42)
    out = dict(lmin=lmin, lmax=lmax, nu=nu, f=f, u_cycles=np.stack(us), rho=rho, rho_steps=steps,
               verts=np.asarray(getattr(tet, "vertices", tet), dtype=float),
               kind=cfg.kind, degrees=np.array(cfg.degrees), variant=cfg.variant)
    # transfers of the top two levels on seeded vectors (bitwise pins of P and P^T)
    P = H.P[top - 1]
    spc = H.spaces[top - 1]
    r = np.where(sp.free, rng.standard_normal(sp.ndof), 0.0)
    rc = P.T @ r
    rc[~spc.free] = 0.0
    e = np.where(spc.free, rng.standard_normal(spc.ndof), 0.0)
    pe = P @ e
    pe[~sp.free] = 0.0
    out.update(xfer_r=r, xfer_rc=rc, xfer_e=e, xfer_pe=pe)
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **out)
    print(name, "rho", rho, "|u|", [float(np.abs(v).max()) for v in us])


def schur_case():
    """SchurComplement._inner_solve (schur.py:80-100, 'multigrid' inner solver) on cell 0 of the cube mesh."""
    from tetilu.schur import SchurComplement
    mesh = geometry.cube_mesh()
    level = 4
    sc = SchurComplement(mesh, level, inner="multigrid")
    n_int = len(sc._cells[0]["ids"])
    rhs = np.random.default_rng(3).standard_normal(n_int)
    x = sc._inner_solve(0, rhs)
    np.savez_compressed(os.path.join(OUT, "schur_inner_L4.npz"), level=level, rhs=rhs, x=x,
                        verts=mesh.cell_tet(0).vertices, inner_tol=sc.inner_tol,
                        degrees=np.array(sc.inner_smoother.degrees), kind=sc.inner_smoother.kind,
                        variant=sc.inner_smoother.variant)
    print("schur inner", n_int, float(np.abs(x).max()))


if __name__ == "__main__":
    schur_case()
    case("mg_unit_L5_surr", UNIT, CoefficientField.constant(1.0), 2, 5,
         SmootherConfig(kind="surrogate_ilu", degrees=(3, 3, 3), variant="v1"), 2)
    case("mg_unit_L5_ilu", UNIT, CoefficientField.constant(1.0), 2, 5, SmootherConfig(kind="ilu"), 1)
    case("mg_dist_L5_surr", DISTORTED, diag_tensor((1, 1, 1e-1)), 3, 5,
         SmootherConfig(kind="surrogate_ilu", degrees=(2, 2, 2), variant="v2"), 2)

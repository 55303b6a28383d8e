"""Convergence factor of the reference V-cycle at level 6 (unit tet, (3,3,3) surrogate smoother, nu = 2 + 2):
the UNMODIFIED reference Hierarchy.convergence_factor, build container only -> tests/golden/mgrho_unit_L6.npz."""
import os, sys, time
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
sys.path.insert(0, "/root/reference/pkg/src")
import numpy as np
from tetilu import geometry
from tetilu.assembly import CoefficientField
from tetilu.multigrid import Hierarchy, SmootherConfig
t=time.time()
mesh = geometry.single_tet_mesh(geometry.trirect_tet(1.0))
H = Hierarchy(mesh, lmin=2, lmax=6, coeff=CoefficientField.constant(1.0), smoother=SmootherConfig(kind="surrogate_ilu", degrees=(3,3,3), variant="v1"), nu_pre=2, nu_post=2)
rho = H.convergence_factor(steps=8, seed=42)
print("L6 rho", rho, time.time()-t)
np.savez_compressed("/root/repo/tests/golden/mgrho_unit_L6.npz", lmin=2, lmax=6, nu=2, rho=rho, rho_steps=8, kind="surrogate_ilu", degrees=np.array((3,3,3)), variant="v1", verts=geometry.trirect_tet(1.0))

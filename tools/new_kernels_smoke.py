"""Small invocations of the setup / multigrid / interface kernels (levels 3-5) for compute-sanitizer or the
bounds-checked build: factorization (constant, per-point, on-the-fly rows), transfers, one V-cycle."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_15280_b200 import SmootherConfig, lattice  # noqa: E402
from paper_2210_15280_b200 import fitting as F  # noqa: E402
from paper_2210_15280_b200 import multigrid as MG  # noqa: E402
from paper_2210_15280_b200 import stencil as S  # noqa: E402

for level in (3, 4, 5):
    for src in (S.stencil_source(lattice.unit_tet(), level, S.CoefficientField.constant(1.0)),
                S.stencil_source(lattice.distorted_tet(), level, S.diag_tensor((1, 1, 1e-3))),
                S.stencil_source(lattice.unit_tet(), level, S.sin_kappa())):
        a = F.factorize_tet(src, level, collect_ranks=lattice.band_ranks(level))
        b = F.factorize_tet_device(src, level, collect_ranks=lattice.band_ranks(level))
        assert np.array_equal(a.rows, b.rows) and np.array_equal(a.collected, b.collected)
H = MG.Hierarchy(lattice.unit_tet(), 2, 5, None, SmootherConfig(degrees=(2, 2, 2)), 1, 1, factorize="device")
g = lattice.grid_size(5)
f = torch.as_tensor(np.where(lattice.interior_mask(5), np.random.default_rng(0).standard_normal(g), 0.0), device="cuda")
u = H.zero(H.top)
H.v_cycle(H.top, u, f)
torch.cuda.synchronize()
print("new kernels ok", float(u.abs().max()))

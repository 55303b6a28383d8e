"""Parity at BASELINE.json's full sizes: the CUDA path against the C oracle (bitwise, exact mode).

* config 4: all 384 Kuhn macro-tets at level 7 (128M DoF), q = 6, through the bench's resident
  packed path (MacroMeshSmoother.load / sweep / store), 2 sweeps, plus the per-sweep norms;
* config 2: the distorted macro-tet with K = diag(1, 1, 1e-3) at level 7 (per-point stencil rows),
  q = 6, 3 sweeps through SurrogateILUSmoother.apply.

Config 1 runs at full size in test_gpu_parity.py (golden vectors); configs 3 and 5 are covered at
reduced levels there (their full-size setup takes tens of minutes on the host).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from paper_2210_15280_b200 import MacroMeshSmoother, SmootherConfig, SurrogateILUSmoother, lattice, stencil  # noqa: E402

pytestmark = pytest.mark.gpu


def _surrogate(sm):
    p = sm.precond
    return O.OracleSurrogate(p.level, p.lcoefs, p.dcoefs, p.variant, p.band_ranks, p.store_rows)


def test_config4_full_384_tets_level7_bitwise():
    level, sweeps = 7, 2
    tets = lattice.kuhn_mesh(4)
    assert len(tets) == 384
    mm = MacroMeshSmoother(tets, level, degrees=(6, 6, 6))
    assert len(mm.groups) == 1          # all Kuhn stencils identical: one shared surrogate
    mask = lattice.interior_mask(level)
    rng = np.random.default_rng(4)
    u0 = np.zeros((len(tets), mask.size))
    u0[:, mask] = rng.uniform(-1.0, 1.0, (len(tets), int(mask.sum())))
    u = torch.as_tensor(u0, device="cuda")
    f = torch.zeros_like(u)
    mm.load(u, f)
    norms = mm.sweep(sweeps)
    mm.store(u)
    sm = mm.smoothers[0]
    sur, arow = _surrogate(sm), np.atleast_1d(sm.source.data)
    ref, zero = u0.copy(), np.zeros_like(u0)
    ref_norms = []
    for _ in range(sweeps):
        # global ||f - A u||^2 before the sweep, summed over all tets (the allreduced quantity)
        ref_norms.append(sum(float(np.dot(r, r)) for r in
                             (-O.stencil_apply(level, arow, ref[t]) for t in range(len(tets)))))
        O.sweeps_many(sur, level, arow, ref, zero, 1)
    assert np.array_equal(u.cpu().numpy(), ref)
    np.testing.assert_allclose(norms.cpu().numpy(), ref_norms, rtol=1e-12)


def test_config2_full_distorted_level7_bitwise():
    level, sweeps = 7, 3
    src = stencil.stencil_source(lattice.distorted_tet(), level, stencil.diag_tensor((1.0, 1.0, 1e-3)))
    assert not src.constant
    sm = SurrogateILUSmoother(src, level, SmootherConfig("surrogate_ilu", (6, 6, 6), "v1"))
    mask = lattice.interior_mask(level)
    u0 = np.zeros(mask.size)
    u0[mask] = np.random.default_rng(2).uniform(-1.0, 1.0, int(mask.sum()))
    f = np.zeros_like(u0)
    u = torch.as_tensor(u0, device="cuda")
    sm.apply(u, torch.zeros_like(u), sweeps)
    ref = u0.copy()
    O.sweeps(_surrogate(sm), level, src.data, ref, f, sweeps)
    assert np.array_equal(u.cpu().numpy(), ref)

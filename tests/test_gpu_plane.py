"""GPU parity of the plane-layout single-tet kernels (tilu_plane.cu) against the C oracle.

Bar: bitwise (np.array_equal) in exact mode; <= 1e-12 max relative error per sweep in fast (FMA)
mode.  Levels 3..7 cover one band / one chunk, partial bands and chunks, several chunks per
diagonal (level 7: up to 4 chunks of 32 rows) and dead warps at the tet's top.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from paper_2210_15280_b200 import DevicePlan, lattice  # noqa: E402
from paper_2210_15280_b200 import fitting as F  # noqa: E402
from paper_2210_15280_b200 import stencil as S  # noqa: E402

pytestmark = pytest.mark.gpu


def cuda(a):
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda")


def relerr(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def case(level, q, variant="v1", coeff=None, verts=None, seed=0, fseed=None):
    verts = lattice.unit_tet() if verts is None else verts
    src = S.stencil_source(verts, level, coeff or S.CoefficientField.constant(1.0))
    fit = F.fit_surrogate_ilu(src, level, (q, q, q), variant)
    mask = lattice.interior_mask(level)
    rng = np.random.default_rng(seed)
    u0 = np.zeros(lattice.grid_size(level))
    u0[mask] = rng.uniform(-1, 1, int(mask.sum()))
    f = np.zeros_like(u0)
    if fseed is not None:
        f[mask] = np.random.default_rng(fseed).normal(size=int(mask.sum()))
    return src, fit, u0, f


def plane_plan(level, src, fit, variant, fast=False, schedule="plane"):
    op = {"arow": src.data} if src.constant else {"arows": src.data}
    return DevicePlan(level, fit.lcoefs, fit.dcoefs, variant, fit.band_ranks, fit.store_rows, fast=fast,
                      schedule=schedule, **op)


def oracle_sweeps(level, src, fit, variant, u0, f, k):
    ref = u0.copy()
    nr = O.sweeps(O.OracleSurrogate(level, fit.lcoefs, fit.dcoefs, variant, fit.band_ranks, fit.store_rows),
                  level, src.data, ref, f, k, return_norms=True)
    return ref, nr


@pytest.mark.parametrize("level,q,variant", [(3, 2, "v1"), (4, 4, "v2"), (5, 4, "v1"), (5, 0, "v1"), (5, 1, "v2"),
                                             (6, 3, "v1"), (6, 6, "v2"), (7, 6, "v1")])
def test_plane_bitwise_vs_oracle(level, q, variant):
    src, fit, u0, f = case(level, q, variant, fseed=level)
    ref, nr = oracle_sweeps(level, src, fit, variant, u0, f, 3)
    p = plane_plan(level, src, fit, variant)
    u = cuda(u0)
    rn = p.sweep(u, cuda(f), 3, norms=True)
    assert np.array_equal(u.cpu().numpy(), ref)
    np.testing.assert_allclose(rn.cpu().numpy().ravel(), nr, rtol=1e-12)


@pytest.mark.parametrize("level,q", [(5, 4), (7, 6)])
def test_plane_fast_mode_within_1e12(level, q):
    src, fit, u0, f = case(level, q)
    sur = O.OracleSurrogate(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows)
    p = plane_plan(level, src, fit, "v1", fast=True)
    u, ref = cuda(u0), u0.copy()
    for _ in range(4):
        O.sweeps(sur, level, src.data, ref, f, 1)
        p.sweep(u, cuda(f), 1)
        assert relerr(u.cpu().numpy(), ref) <= 1e-12


def test_plane_per_point_stencil_config2_geometry():
    """Tensor coefficient on the distorted tet (configs 2/5): per-point stencil rows."""
    level = 5
    src, fit, u0, f = case(level, 4, "v1", coeff=S.diag_tensor((1.0, 1.0, 1e-3)), verts=lattice.distorted_tet(),
                           seed=2)
    assert not src.constant
    ref, _ = oracle_sweeps(level, src, fit, "v1", u0, f, 2)
    u = cuda(u0)
    plane_plan(level, src, fit, "v1").sweep(u, cuda(f), 2)
    assert np.array_equal(u.cpu().numpy(), ref)


def test_plane_state_across_calls_and_plans():
    """The plan's plane workspace (armed handoff positions) stays consistent across calls, and
    results equal one multi-sweep call and the other schedules."""
    level, q = 6, 4
    src, fit, u0, f = case(level, q, fseed=3)
    p = plane_plan(level, src, fit, "v1")
    u1 = cuda(u0)
    p.sweep(u1, cuda(f), 4)
    u2 = cuda(u0)
    for _ in range(4):
        p.sweep(u2, cuda(f), 1)
    u3 = cuda(u0)
    plane_plan(level, src, fit, "v1", schedule="batch").sweep(u3, cuda(f), 4)
    assert np.array_equal(u1.cpu().numpy(), u2.cpu().numpy())
    assert np.array_equal(u1.cpu().numpy(), u3.cpu().numpy())


def test_plane_boundary_untouched():
    level = 5
    src, fit, u0, f = case(level, 4)
    mask = lattice.interior_mask(level)
    u0b = u0.copy()
    u0b[~mask] = 0.0
    u = cuda(u0b)
    plane_plan(level, src, fit, "v1").sweep(u, cuda(f), 2)
    assert np.all(u.cpu().numpy()[~mask] == 0.0)


@pytest.mark.parametrize("level", [5, 7])
def test_plane_stored_factor_sweep_bitwise(level):
    """CellILU (stored ILU(0) factors, ilu.py:210-227) through the plane kernels: the march helpers
    read the factor rows instead of marching surrogates."""
    src, fit, u0, f = case(level, 4, fseed=11)
    fr = F.factorize_tet(src, level, full_store=True)
    ref = u0.copy()
    O.sweeps(None, level, src.data, ref, f, 3, factors=fr.rows)
    p = DevicePlan(level, np.zeros((7, 1, 1, 1)), np.zeros(1), "v2", factors=fr.rows, arow=src.data,
                   schedule="plane")
    u = cuda(u0)
    p.sweep(u, cuda(f), 3, stored=True)
    assert np.array_equal(u.cpu().numpy(), ref)


def test_plane_config3_variable_coefficient():
    """Config 3's coefficient k(x) = 1 + 0.5 sin(2 pi x) sin(2 pi y) sin(2 pi z) (per-point stencil
    rows, f ~ N(0, 1), u = 0) through the plane kernels, bitwise vs the oracle."""
    level = 6
    src, fit, _, f = case(level, 6, "v1", coeff=S.sin_kappa(), fseed=3)
    assert not src.constant
    u0 = np.zeros_like(f)
    ref, nr = oracle_sweeps(level, src, fit, "v1", u0, f, 3)
    u = cuda(u0)
    rn = plane_plan(level, src, fit, "v1").sweep(u, cuda(f), 3, norms=True)
    assert np.array_equal(u.cpu().numpy(), ref)
    np.testing.assert_allclose(rn.cpu().numpy().ravel(), nr, rtol=1e-12)


def test_plane_level8_eight_chunks_bitwise():
    """Level 8: diagonals of up to 253 rows (8 chunks of 32), 64 bands -- the cross-chunk and
    cross-band handoffs at the scale of the level-9 runs."""
    level = 8
    src, fit, u0, f = case(level, 6, "v1", fseed=8)
    ref, nr = oracle_sweeps(level, src, fit, "v1", u0, f, 2)
    u = cuda(u0)
    rn = plane_plan(level, src, fit, "v1").sweep(u, cuda(f), 2, norms=True)
    assert np.array_equal(u.cpu().numpy(), ref)
    np.testing.assert_allclose(rn.cpu().numpy().ravel(), nr, rtol=1e-12)


def test_plane_two_streams_share_a_plan():
    """Calls on two streams sharing one plan (and its plane workspace) serialise correctly."""
    level = 6
    src, fit, u0, f = case(level, 4, fseed=5)
    p = plane_plan(level, src, fit, "v1")
    ref = cuda(u0)
    p.sweep(ref, cuda(f), 3)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    ua, ub = cuda(u0), cuda(u0 * 0.5)
    fa, fb = cuda(f), cuda(f * 0.5)
    torch.cuda.synchronize()
    with torch.cuda.stream(s1):
        p.sweep(ua, fa, 3)
    with torch.cuda.stream(s2):
        p.sweep(ub, fb, 3)
    torch.cuda.synchronize()
    assert np.array_equal(ua.cpu().numpy(), ref.cpu().numpy())
    ref_b = cuda(u0 * 0.5)
    p.sweep(ref_b, cuda(f * 0.5), 3)
    assert np.array_equal(ub.cpu().numpy(), ref_b.cpu().numpy())

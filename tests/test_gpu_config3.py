"""Config 3 (variable coefficient k(x) = 1 + 0.5 sin sin sin on the unit tet) on the GPU with the
operator rows evaluated on the fly from the separable tables (stencil.SeparableK): no per-point rows
on the device.  Bar: bitwise vs the C oracle fed the reference-equal per-point rows (exact mode),
<= 1e-12 per sweep in fast (FMA) mode; at level 9 (the north star's size) against the committed
oracle fixture tests/golden/l9_config3.npz (SHA-256 of the full u after sweeps 1, 2, 3, 100)."""
import hashlib
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from conftest import GOLDEN  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2210_15280_b200 import DevicePlan, SurrogateILUSmoother, lattice  # noqa: E402
from paper_2210_15280_b200 import fitting as F  # noqa: E402
from paper_2210_15280_b200 import stencil as S  # noqa: E402

pytestmark = pytest.mark.gpu


def cuda(a):
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda")


def relerr(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def setup(level, q, variant="v1", fseed=3):
    src = S.stencil_source(lattice.unit_tet(), level, S.sin_kappa())
    assert src.sepk is not None
    fit = F.fit_surrogate_ilu(src, level, (q, q, q), variant)
    mask = lattice.interior_mask(level)
    f = np.zeros(lattice.grid_size(level))
    f[mask] = np.random.default_rng(fseed).normal(size=int(mask.sum()))
    return src, fit, f


def sepk_plan(level, src, fit, variant, **kw):
    return DevicePlan(level, fit.lcoefs, fit.dcoefs, variant, fit.band_ranks, fit.store_rows, sepk=src.sepk, **kw)


@pytest.mark.parametrize("level,q,variant,schedule", [
    (4, 4, "v1", "simple"), (4, 3, "v1", "plane"), (5, 4, "v1", "auto"), (5, 4, "v2", "auto"),
    (6, 6, "v1", "auto"), (7, 6, "v1", "auto"), (8, 6, "v1", "auto")])
def test_sepk_sweeps_bitwise_vs_oracle(level, q, variant, schedule):
    src, fit, f = setup(level, q, variant)
    u0 = np.zeros_like(f)
    ref = u0.copy()
    nr = O.sweeps(O.OracleSurrogate(level, fit.lcoefs, fit.dcoefs, variant, fit.band_ranks, fit.store_rows),
                  level, src.data, ref, f, 3, return_norms=True)
    u = cuda(u0)
    rn = sepk_plan(level, src, fit, variant, schedule=schedule).sweep(u, cuda(f), 3, norms=True)
    assert np.array_equal(u.cpu().numpy(), ref)
    np.testing.assert_allclose(rn.cpu().numpy().ravel(), nr, rtol=1e-12)


@pytest.mark.parametrize("level", [5, 7])
def test_sepk_fast_mode_within_1e12(level):
    src, fit, f = setup(level, 6)
    sur = O.OracleSurrogate(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows)
    p = sepk_plan(level, src, fit, "v1", fast=True)
    ref = np.zeros_like(f)
    u = cuda(ref)
    for _ in range(4):
        O.sweeps(sur, level, src.data, ref, f, 1)
        p.sweep(u, cuda(f), 1)
        assert relerr(u.cpu().numpy(), ref) <= 1e-12


@pytest.mark.parametrize("level", [4, 6])
def test_sepk_residual_and_stencil_apply_bitwise(level):
    src, fit, f = setup(level, 4)
    mask = lattice.interior_mask(level)
    u0 = np.zeros_like(f)
    u0[mask] = np.random.default_rng(1).uniform(-1, 1, int(mask.sum()))
    p = sepk_plan(level, src, fit, "v1")
    out = p.stencil_apply(cuda(u0)).cpu().numpy()
    want = O.stencil_apply(level, src.data, u0)
    assert np.array_equal(out[mask], want[mask])
    w, rn = p.residual(cuda(u0), cuda(f), norms=True)
    r = np.where(mask, f - want, 0.0)
    assert np.array_equal(w.cpu().numpy(), r)
    np.testing.assert_allclose(float(rn[0]), float(np.sum(r ** 2)), rtol=1e-12)


def test_smoother_api_uses_the_table_form():
    """SurrogateILUSmoother.setup(unit tet, coeff=sin_kappa()) builds a plan without per-point rows
    and equals the oracle bitwise."""
    level = 6
    sm = SurrogateILUSmoother.setup(lattice.unit_tet(), level, (6, 6, 6), coeff=S.sin_kappa())
    assert sm.source.sepk is not None and not hasattr(sm.plan, "_arows")
    mask = lattice.interior_mask(level)
    f = np.zeros(lattice.grid_size(level))
    f[mask] = np.random.default_rng(3).normal(size=int(mask.sum()))
    u = torch.zeros(lattice.grid_size(level), dtype=torch.float64, device="cuda")
    rn = sm.apply(u, cuda(f), 2, residual_norms=True)
    pre = sm.precond
    ref = np.zeros_like(f)
    nr = O.sweeps(O.OracleSurrogate(level, pre.lcoefs, pre.dcoefs, "v1", pre.band_ranks, pre.store_rows), level,
                  sm.source.data, ref, f, 2, return_norms=True)
    assert np.array_equal(u.cpu().numpy(), ref)
    np.testing.assert_allclose(rn.cpu().numpy().ravel(), nr, rtol=1e-12)


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def l9():
    path = os.path.join(GOLDEN, "l9_config3.npz")
    if not os.path.exists(path):
        pytest.skip("l9_config3.npz not generated (tests/golden/make_config3_l9.py)")
    g = np.load(path)
    level = int(g["level"])
    sk = S.SeparableK(level, g["tables"], float(g["c0"]), float(g["w"]))
    rows = sk.rows()                                    # native builder, same rows as the fixture's
    assert _sha(rows) == str(g["rows_sha"])
    src = S.StencilSource(level, rows, False, sk)
    band = lattice.band_ranks(level)
    fr = F.factorize_tet(src, level, full_store=False, collect_ranks=band)  # deterministic native LDL^T
    assert _sha(fr.collected) == str(g["band_sha"])
    mask = lattice.interior_mask(level)
    f = np.zeros(lattice.grid_size(level))
    f[mask] = np.random.default_rng(int(g["fseed"])).normal(size=int(mask.sum()))
    return g, sk, band, fr.collected, f


@pytest.mark.parametrize("fast", [False, True])
def test_config3_level9_vs_oracle_fixture(l9, fast):
    """The full configs[2] run: level 9 (22.1M DoF), 100 sweeps, residual norm before every sweep
    and after the last one.  Exact mode: the full u is bitwise the oracle's after sweeps 1, 2, 3
    and 100 (SHA-256); fast mode: <= 1e-12 relative at the sampled points after every snapshot."""
    g, sk, band, store, f = l9
    level = int(g["level"])
    p = DevicePlan(level, g["lcoefs"], g["dcoefs"], "v1", band, store, sepk=sk, fast=fast)
    u = torch.zeros(lattice.grid_size(level), dtype=torch.float64, device="cuda")
    fd = cuda(f)
    snaps = list(g["snaps"])
    norms, done = [], 0
    for i, k in enumerate(snaps):
        rn = p.sweep(u, fd, k - done, norms=True)
        norms.append(rn.cpu().numpy().ravel())
        done = k
        uh = u.cpu().numpy()
        if fast:
            got, want = uh[g["sample_ranks"]], g["u_sample"][i]
            assert relerr(got, want) <= 1e-12, (k, relerr(got, want))
        else:
            assert _sha(uh) == str(g["u_sha"][i]), f"u after sweep {k} differs from the oracle"
    w, rfin = p.residual(u, fd, norms=True)
    norms = np.concatenate(norms)
    np.testing.assert_allclose(norms, g["rnorm2"], rtol=1e-10 if fast else 1e-12)
    np.testing.assert_allclose(float(rfin[0]), float(g["rnorm2_final"]), rtol=1e-10 if fast else 1e-12)
    # the smoother converges: residual decreases monotonically after the first sweeps
    assert g["rnorm2"][-1] < g["rnorm2"][1]

"""API guards and routing on the GPU (advisor findings, round 1):
* operator-surrogate plans (a_mode='surrogate') at level >= 6 and for batches must not reach the
  batched kernels (they have no surrogate residual) -- they run and match the oracle;
* kind='ilu' uses the assembled operator even when a_mode='surrogate' (reference multigrid.py:418);
* mismatched batch shapes / devices raise instead of reading past an allocation."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from paper_2210_15280_b200 import DevicePlan, SurrogateILUSmoother, lattice  # noqa: E402
from paper_2210_15280_b200 import fitting as F  # noqa: E402
from paper_2210_15280_b200 import stencil as S  # noqa: E402

pytestmark = pytest.mark.gpu


def cuda(a):
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda")


def u0_of(level, ntets=1, seed=0):
    mask = lattice.interior_mask(level)
    rng = np.random.default_rng(seed)
    u = np.zeros((ntets, lattice.grid_size(level)))
    for t in range(ntets):
        u[t, mask] = rng.uniform(-1, 1, int(mask.sum()))
    return u


@pytest.mark.parametrize("level,ntets", [(6, 1), (4, 2), (5, 3)])
def test_operator_surrogate_plan_routes_safely(level, ntets):
    src = S.stencil_source(lattice.unit_tet(), level, S.sin_kappa())
    fit = F.fit_surrogate_ilu(src, level, (4, 4, 4), "v1")
    ac = F.fit_surrogate_operator(src, level, (3, 3, 3))
    p = DevicePlan(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows, acoefs=ac)
    u0 = u0_of(level, ntets)
    f = np.zeros_like(u0)
    u = cuda(u0)
    p.sweep(u, cuda(f), 2)
    sur = O.OracleSurrogate(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows)
    for t in range(ntets):
        ref = u0[t].copy()
        O.sweeps(sur, level, None, ref, f[t], 2, acoefs=ac)
        assert np.array_equal(u[t].cpu().numpy(), ref)


def test_ilu_kind_ignores_operator_surrogate():
    level = 5
    cfg = dict(kind="ilu", a_mode="surrogate", a_degrees=(2, 2, 2))
    sm = SurrogateILUSmoother.setup(lattice.unit_tet(), level, (4, 4, 4), coeff=S.sin_kappa(), **cfg)
    assert sm.plan is not None
    u0 = u0_of(level)[0]
    f = np.zeros_like(u0)
    u = cuda(u0)
    sm.apply(u, cuda(f), 2)
    ref = u0.copy()
    O.sweeps(None, level, sm.source.data, ref, f, 2, factors=sm.factorization.rows)
    assert np.array_equal(u.cpu().numpy(), ref)


def test_batch_shape_mismatch_raises():
    level = 4
    src = S.stencil_source(lattice.unit_tet(), level, S.CoefficientField.constant(1.0))
    fit = F.fit_surrogate_ilu(src, level, (3, 3, 3), "v1")
    p = DevicePlan(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows, arow=src.data)
    g = lattice.grid_size(level)
    u2 = torch.zeros((2, g), dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        p.sweep(u2, torch.zeros(g, dtype=torch.float64, device="cuda"), 1)
    with pytest.raises(ValueError):
        p.residual(u2, torch.zeros((3, g), dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        p.pack(u2, ntets=3)
    with pytest.raises(ValueError):
        p.stencil_apply(u2, out=torch.zeros((1, g), dtype=torch.float64, device="cuda"))


@pytest.mark.parametrize("level,ntets,fast", [(5, 40, False), (7, 2, False), (6, 3, True)])
def test_operator_surrogate_batched_kernels(level, ntets, fast):
    """a_mode='surrogate' through the batched kernels (15 operator-surrogate marchers shared by the
    warp, surrogate_apply_residual order): bitwise vs the oracle (exact), <= 1e-12 (fast); 40 tets
    take two-tet lanes (T = 2)."""
    src = S.stencil_source(lattice.unit_tet(), level, S.sin_kappa())
    fit = F.fit_surrogate_ilu(src, level, (4, 4, 4), "v1")
    ac = F.fit_surrogate_operator(src, level, (3, 3, 3))
    p = DevicePlan(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows, acoefs=ac, fast=fast)
    u0 = u0_of(level, ntets, seed=7)
    f = np.zeros_like(u0)
    f[:, lattice.interior_mask(level)] = 0.25
    u = cuda(u0)
    rn = p.sweep(u, cuda(f), 2, norms=True)
    sur = O.OracleSurrogate(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows)
    got = u.cpu().numpy()
    for t in range(ntets):
        ref = u0[t].copy()
        nr = O.sweeps(sur, level, None, ref, f[t], 2, acoefs=ac, return_norms=True)
        if fast:
            assert float(np.abs(got[t] - ref).max() / np.abs(ref).max()) <= 1e-12
        else:
            assert np.array_equal(got[t], ref)
        np.testing.assert_allclose(rn.cpu().numpy()[:, t], nr, rtol=1e-10 if fast else 1e-12)


@pytest.mark.parametrize("level,ntets,stored", [(5, 1, False), (6, 1, False), (7, 1, False), (5, 3, False), (6, 40, False),
                                                (6, 1, True)])
def test_solve_into_fast_route_equals_reference_layout_kernels(level, ntets, stored):
    """The drop-in solve_into runs on the plane / batched sweep kernels (one step from u = 0 with a zero
    operator row: r = f exactly); it must equal the reference-layout wavefront kernels bit for bit, with or
    without an operator on the plan."""
    src = S.stencil_source(lattice.distorted_tet(), level, S.diag_tensor((1, 1e-2, 1)))
    mask = lattice.interior_mask(level)
    w0 = np.zeros((ntets, lattice.grid_size(level)))
    w0[:, mask] = np.random.default_rng(level).standard_normal((ntets, int(mask.sum())))
    outs = []
    if stored:
        fac = F.factorize_tet(src, level).rows
        z = np.zeros((7, 1, 1, 1))
        for sched in ("auto", "simple"):
            p = DevicePlan(level, z, np.zeros(1), "v2", factors=fac, schedule=sched)
            w = cuda(w0[0])
            p.stored_solve_into(w)
            outs.append(w.cpu().numpy())
    else:
        fit = F.fit_surrogate_ilu(src, level, (3, 3, 3), "v1")
        for sched, op in (("auto", {}), ("auto", {"arows": src.data}), ("simple", {})):
            p = DevicePlan(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows, schedule=sched, **op)
            w = cuda(w0 if ntets > 1 else w0[0])
            p.solve_into(w)
            outs.append(w.cpu().numpy())
    for o in outs[:-1]:
        assert np.array_equal(o, outs[-1])
    assert not np.any(outs[0].reshape(ntets, -1)[:, ~mask])


@pytest.mark.parametrize("level,adeg,fast", [(5, (3, 3, 3), False), (7, (2, 2, 2), False), (7, (3, 3, 3), False),
                                             (6, (1, 1, 1), False), (6, (3, 3, 3), True)])
def test_operator_surrogate_in_plane_kernels(level, adeg, fast):
    """a_mode='surrogate' on one macro-tet from level 5 up runs in the plane kernels' residual helper
    (15 marched tables in registers); bitwise vs the oracle's surrogate_apply_residual sweep, the fast (FMA)
    mode within 1e-12."""
    src = S.stencil_source(lattice.unit_tet(), level, S.sin_kappa())
    fit = F.fit_surrogate_ilu(src, level, (4, 4, 4), "v1")
    ac = F.fit_surrogate_operator(src, level, adeg)
    p = DevicePlan(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows, acoefs=ac, fast=fast)
    u0 = u0_of(level)[0]
    f = np.zeros_like(u0)
    f[lattice.interior_mask(level)] = np.random.default_rng(2).standard_normal(lattice.interior_size(level))
    u = cuda(u0)
    rn = p.sweep(u, cuda(f), 3, norms=True)
    sur = O.OracleSurrogate(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows)
    ref = u0.copy()
    O.sweeps(sur, level, None, ref, f, 3, acoefs=ac)
    got = u.cpu().numpy()
    if fast:
        assert float(np.abs(got - ref).max() / np.abs(ref).max()) <= 1e-12
    else:
        assert np.array_equal(got, ref)
    assert rn.shape == (3, 1) and np.all(np.isfinite(rn.cpu().numpy()))


@pytest.mark.parametrize("level", [4, 5, 6])
@pytest.mark.parametrize("sched", ["simple", "plane", "batch", "auto"])
@pytest.mark.parametrize("ntets", [1, 3])
def test_boundary_values_are_read_as_given(level, sched, ntets):
    """The cell stage of a hybrid mesh hands tets whose boundary entries carry the shared interface values
    (multigrid.py:414-429): every kernel family reads them in the residual and never writes them."""
    src = S.stencil_source(lattice.distorted_tet(), level, S.diag_tensor((1, 1, 1e-1)))
    fit = F.fit_surrogate_ilu(src, level, (3, 3, 3), "v1")
    g = lattice.grid_size(level)
    mask = lattice.interior_mask(level)
    rng = np.random.default_rng(level)
    u0 = rng.uniform(-1, 1, g)
    f = np.where(mask, rng.standard_normal(g), 0.0)
    ref = u0.copy()
    O.sweeps(O.OracleSurrogate(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows), level, src.data, ref, f, 2)
    p = DevicePlan(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows, arows=src.data, schedule=sched)
    u = cuda(np.tile(u0, (ntets, 1)) if ntets > 1 else u0)
    p.sweep(u, cuda(np.tile(f, (ntets, 1)) if ntets > 1 else f), 2)
    got = u.cpu().numpy().reshape(ntets, -1)
    for t in range(ntets):
        assert np.array_equal(got[t], ref)
    # a later all-Dirichlet call on the same plan must not see the old boundary values (the planes persist)
    z0 = np.where(mask, u0, 0.0)
    ref0 = z0.copy()
    O.sweeps(O.OracleSurrogate(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows), level, src.data, ref0, f, 1)
    u = cuda(z0)
    p.sweep(u, cuda(f), 1)
    assert np.array_equal(u.cpu().numpy(), ref0)


def test_check_finite_reports_a_corrupted_iterate():
    level = 5
    sm = SurrogateILUSmoother.setup(lattice.unit_tet(), level, (3, 3, 3))
    u = cuda(u0_of(level)[0])
    f = torch.zeros_like(u)
    rn = sm.apply(u, f, 2, check_finite=True)
    assert rn.shape == (2, 1)
    u[int(np.nonzero(lattice.interior_mask(level))[0][100])] = float("nan")
    with pytest.raises(FloatingPointError):
        sm.apply(u, f, 1, check_finite=True)


@pytest.mark.parametrize("ntets", [33, 70, 96, 97])
def test_batch_group_shapes_bitwise(ntets):
    """Tets-per-lane selection (one tet per lane up to 32 and for 65..96 tets, two otherwise): partly filled
    groups and both group widths give the oracle's result for every tet."""
    level = 4
    src = S.stencil_source(lattice.kuhn_tet((0, 1, 2)), level, S.CoefficientField.constant(1.0))
    fit = F.fit_surrogate_ilu(src, level, (3, 3, 3), "v1")
    p = DevicePlan(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows, arow=src.data)
    u0 = u0_of(level, ntets, seed=ntets)
    f = np.zeros_like(u0)
    u = cuda(u0)
    p.sweep(u, cuda(f), 2)
    got = u.cpu().numpy()
    sur = O.OracleSurrogate(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows)
    for t in (0, 31, 32, ntets - 1):
        ref = u0[t].copy()
        O.sweeps(sur, level, src.data, ref, f[t], 2)
        assert np.array_equal(got[t], ref), t

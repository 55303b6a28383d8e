"""GPU parity: the CUDA path (through the C ABI) against the C oracle / golden vectors.

Bar: bitwise in the default exact mode (same operation order, no FMA), <= 1e-12 max
relative error per sweep in fast (FMA) mode, asymptotic rate to 3 significant digits.
"""

import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from paper_2210_15280_b200 import (DevicePlan, SurrogateILUSmoother, build_surrogate_ilu,  # noqa: E402
                                   lattice)
from paper_2210_15280_b200 import fitting as F  # noqa: E402
from paper_2210_15280_b200 import stencil as S  # noqa: E402

pytestmark = pytest.mark.gpu
CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "cfg*.npz")))
DEV = "cuda"


def load(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def plan_of(d, fast=False, simple=False, **op):
    return DevicePlan(int(d["level"]), d["lcoefs"], d["dcoefs"], str(d["variant"]), d["band_ranks"],
                      d["store_rows"], fast=fast, simple=simple, **op)


def op_of(d):
    a = d["arows"]
    return {"arow": a[0]} if a.shape[0] == 1 else {"arows": a}


def cuda(a):
    return torch.as_tensor(np.ascontiguousarray(a), device=DEV)


def relerr(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.mark.parametrize("name", CASES)
def test_solve_into_bitwise_vs_reference(name):
    d = load(name)
    if "solve_in" not in d:
        pytest.skip("no solve pin")
    w = cuda(d["solve_in"])
    plan_of(d).solve_into(w)
    assert np.array_equal(w.cpu().numpy(), d["solve_out"])


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("simple", [True, False])
def test_sweeps_bitwise_vs_reference(name, simple):
    d = load(name)
    k = int(d["sweeps"])
    p = plan_of(d, simple=simple, **op_of(d))
    u, f = cuda(d["u0"]), cuda(d["f"])
    rn = p.sweep(u, f, 1, norms=True)
    assert np.array_equal(u.cpu().numpy(), d["u_after_1"])
    rn2 = p.sweep(u, f, k - 1, norms=True)
    assert np.array_equal(u.cpu().numpy(), d[f"u_after_{k}"])
    norms = np.concatenate([rn.cpu().numpy().ravel(), rn2.cpu().numpy().ravel()])
    np.testing.assert_allclose(norms, d["rnorm2"], rtol=1e-12, atol=1e-300)


@pytest.mark.parametrize("name", ["cfg1_L5_v1", "cfg2_L4_v1"])
def test_stored_ilu_bitwise(name):
    d = load(name)
    p = DevicePlan(int(d["level"]), np.zeros((7, 1, 1, 1)), np.zeros(1), "v2", factors=d["factors"], **op_of(d))
    w = cuda(d["ilu_solve_in"])
    p.stored_solve_into(w)
    assert np.array_equal(w.cpu().numpy(), d["ilu_solve_out"])
    u, f = cuda(d["u0"]), cuda(d["f"])
    p.sweep(u, f, int(d["sweeps"]), stored=True)
    assert np.array_equal(u.cpu().numpy(), d["ilu_u_final"])


@pytest.mark.parametrize("name", ["nddf_L3", "nddf_L4", "nddf_L5"])
@pytest.mark.parametrize("variant", ["v1", "v2"])
def test_random_shapes_bitwise(name, variant):
    d = load(name)
    L = int(d["level"])
    for i, _ in enumerate(d["shapes"]):
        p = DevicePlan(L, d[f"s{i}_lcoefs"], d[f"s{i}_dcoefs"], variant, d["band_ranks"], d[f"s{i}_store"])
        w = cuda(d[f"s{i}_w0"])
        p.forward(w)
        assert np.array_equal(w.cpu().numpy(), d[f"s{i}_{variant}_fwd"])
        p.backward(w)
        assert np.array_equal(w.cpu().numpy(), d[f"s{i}_{variant}_solve"])


def test_stencil_apply_and_operator_surrogate_bitwise():
    d = load("kernels_L4")
    z = np.zeros((7, 1, 1, 1))
    p = DevicePlan(4, z, np.zeros(1), "v2", arows=d["arows"])
    assert np.array_equal(p.stencil_apply(cuda(d["u"])).cpu().numpy(), d["stencil_out"])
    p1 = DevicePlan(4, z, np.zeros(1), "v2", arow=d["arow1"][0])
    assert np.array_equal(p1.stencil_apply(cuda(d["u"])).cpu().numpy(), d["stencil_out1"])
    ps = DevicePlan(4, z, np.zeros(1), "v2", acoefs=d["acoefs"])
    w = ps.residual(cuda(d["u"]), cuda(d["f"]))
    assert np.array_equal(w.cpu().numpy(), d["sres_out"])
    s = load("sop_L4")
    pp = plan_of(s, acoefs=s["acoefs"])
    u = torch.zeros(len(s["f"]), dtype=torch.float64, device=DEV)
    pp.sweep(u, cuda(s["f"]), 3)
    assert np.array_equal(u.cpu().numpy(), s["u_after_3"])


def _oracle_case(level, q, variant="v1", coeff=None, verts=None, seed=0):
    verts = lattice.unit_tet() if verts is None else verts
    src = S.stencil_source(verts, level, coeff or S.CoefficientField.constant(1.0))
    fit = F.fit_surrogate_ilu(src, level, (q, q, q), variant)
    mask = lattice.interior_mask(level)
    u0 = np.zeros(lattice.grid_size(level))
    u0[mask] = np.random.default_rng(seed).uniform(-1, 1, int(mask.sum()))
    return src, fit, u0


@pytest.mark.parametrize("level,q,variant", [(2, 3, "v1"), (3, 2, "v2"), (6, 4, "v1"), (6, 6, "v2"), (7, 6, "v1")])
@pytest.mark.parametrize("simple", [True, False])
def test_larger_levels_bitwise_vs_oracle(level, q, variant, simple):
    src, fit, u0 = _oracle_case(level, q, variant)
    f = np.zeros_like(u0)
    ref = u0.copy()
    O.sweeps(O.OracleSurrogate(level, fit.lcoefs, fit.dcoefs, variant, fit.band_ranks, fit.store_rows),
             level, src.data, ref, f, 3)
    p = DevicePlan(level, fit.lcoefs, fit.dcoefs, variant, fit.band_ranks, fit.store_rows, arow=src.data,
                   simple=simple)
    u = cuda(u0)
    p.sweep(u, cuda(f), 3)
    assert np.array_equal(u.cpu().numpy(), ref)


@pytest.mark.parametrize("simple", [True, False])
def test_fast_mode_within_1e12(simple):
    level, q = 6, 4
    src, fit, u0 = _oracle_case(level, q)
    f = np.zeros_like(u0)
    sur = O.OracleSurrogate(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows)
    p = DevicePlan(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows, arow=src.data, fast=True,
                   simple=simple)
    u, ref = cuda(u0), u0.copy()
    for _ in range(5):
        O.sweeps(sur, level, src.data, ref, f, 1)
        p.sweep(u, cuda(f), 1)
        assert relerr(u.cpu().numpy(), ref) <= 1e-12


@pytest.mark.parametrize("simple", [True, False])
def test_batched_tets_equal_single(simple):
    """A batch [T, grid] sharing one surrogate equals T independent sweeps (config 4 path)."""
    level, q = 5, 6
    src, fit, u0 = _oracle_case(level, q, verts=lattice.kuhn_tet((0, 1, 2)))
    T = 7
    rng = np.random.default_rng(5)
    us = np.stack([u0 * s for s in rng.uniform(0.5, 2.0, T)])
    fs = np.zeros_like(us)
    fs[2] = u0
    p = DevicePlan(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows, arow=src.data,
                   simple=simple)
    ub = cuda(us)
    rn = p.sweep(ub, cuda(fs), 2, norms=True)
    sur = O.OracleSurrogate(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows)
    for t in range(T):
        ref = us[t].copy()
        nr = O.sweeps(sur, level, src.data, ref, fs[t], 2, return_norms=True)
        assert np.array_equal(ub[t].cpu().numpy(), ref)
        np.testing.assert_allclose(rn[:, t].cpu().numpy(), nr, rtol=1e-12)


def test_rate_three_digits_config1():
    """configs[0]: L5 unit tet, q=4, 20 sweeps, f=0: last-step ratio equals the reference's
    to 3 significant digits (bitwise in fact)."""
    d = load("cfg1_L5_v1")
    sm = SurrogateILUSmoother.setup(lattice.unit_tet(), 5, (4, 4, 4))
    u = cuda(d["u0"])
    norms = []
    for _ in range(20):
        sm.apply(u, cuda(d["f"]), 1)
        norms.append(float(torch.linalg.norm(u)))
    rho, rho_ref = norms[-1] / norms[-2], d["unorms"][-1] / d["unorms"][-2]
    assert f"{rho:.3g}" == f"{rho_ref:.3g}"
    assert np.array_equal(u.cpu().numpy(), d["u_after_20"])


def test_solve_into_numpy_dropin():
    d = load("cfg1_L5_v2")
    sur = build_surrogate_ilu(S.stencil_source(lattice.unit_tet(), 5, S.CoefficientField.constant(1.0)), 5,
                              (4, 4, 4), "v2")
    w = d["solve_in"].copy()
    sur.solve_into(w)
    assert np.array_equal(w, d["solve_out"])


def test_errors_fail_loudly():
    d = load("cfg1_L5_v1")
    p = plan_of(d, **op_of(d))
    with pytest.raises(ValueError):
        p.solve_into(torch.zeros(len(d["u0"]), dtype=torch.float64))          # CPU tensor
    with pytest.raises(TypeError):
        p.solve_into(torch.zeros(len(d["u0"]), dtype=torch.float32, device=DEV))
    with pytest.raises(ValueError):
        p.solve_into(torch.zeros(len(d["u0"]) + 1, dtype=torch.float64, device=DEV))
    with pytest.raises(Exception):
        DevicePlan(5, d["lcoefs"], d["dcoefs"], "v1", d["band_ranks"][:-1], d["store_rows"][:-1])


@pytest.mark.parametrize("T,level,q,variant", [(40, 5, 6, "v1"), (33, 4, 3, "v2"), (2, 6, 4, "v1")])
def test_packed_batches_bitwise(T, level, q, variant):
    """Interleaved fast path with padding groups (T not a multiple of 32), V1 and V2."""
    src, fit, u0 = _oracle_case(level, q, variant, verts=lattice.kuhn_tet((2, 0, 1)))
    rng = np.random.default_rng(T)
    us = np.stack([u0 * s for s in rng.uniform(-2.0, 2.0, T)])
    fs = np.zeros_like(us)
    mask = lattice.interior_mask(level)
    fs[:, mask] = rng.standard_normal((T, int(mask.sum())))
    p = DevicePlan(level, fit.lcoefs, fit.dcoefs, variant, fit.band_ranks, fit.store_rows, arow=src.data)
    ub = cuda(us)
    rn = p.sweep(ub, cuda(fs), 3, norms=True)
    sur = O.OracleSurrogate(level, fit.lcoefs, fit.dcoefs, variant, fit.band_ranks, fit.store_rows)
    for t in range(T):
        ref = us[t].copy()
        nr = O.sweeps(sur, level, src.data, ref, fs[t], 3, return_norms=True)
        assert np.array_equal(ub[t].cpu().numpy(), ref), t
        np.testing.assert_allclose(rn[:, t].cpu().numpy(), nr, rtol=1e-12)


def test_packed_resident_api_and_roundtrip():
    level, q, T = 5, 4, 37
    src, fit, u0 = _oracle_case(level, q)
    p = DevicePlan(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows, arow=src.data)
    us = cuda(np.stack([u0 * (1 + 0.01 * t) for t in range(T)]))
    back = torch.empty_like(us)
    p.unpack(p.pack(us), back)
    assert torch.equal(back, us)
    up, fp = p.pack(us), p.pack(torch.zeros_like(us))
    wp = p.new_scratch(T)
    p.sweep_packed(up, fp, wp, T, 2)
    ref = us.clone()
    p.sweep(ref, torch.zeros_like(us), 2)     # reference-layout entry point
    p.unpack(up, back)
    assert torch.equal(back, ref)


@pytest.mark.parametrize("T", [3, 70])
def test_packed_scratch_state_across_calls(T):
    """The scratch keeps the sentinel-armed work vectors across calls: k single-sweep calls equal one
    k-sweep call bitwise, and a clobbered scratch (header no longer matching) is re-armed."""
    level, q = 5, 5
    src, fit, u0 = _oracle_case(level, q, verts=lattice.kuhn_tet((2, 1, 0)))
    p = DevicePlan(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows, arow=src.data)
    rng = np.random.default_rng(T)
    us = cuda(np.stack([u0 * s for s in rng.uniform(0.5, 2.0, T)]))
    fs = cuda(rng.standard_normal(us.shape) * lattice.interior_mask(level))
    up1, up3, fp = p.pack(us), p.pack(us), p.pack(fs)
    w1, w3 = p.new_scratch(T), p.new_scratch(T)
    for _ in range(3):
        p.sweep_packed(up1, fp, w1, T, 1)
    p.sweep_packed(up3, fp, w3, T, 3)
    assert torch.equal(up1, up3)
    w1.fill_(1.0)                              # clobber: values, boundary and header
    p.sweep_packed(up1, fp, w1, T, 1)
    p.sweep_packed(up3, fp, w3, T, 1)
    assert torch.equal(up1, up3)


def test_packed_fast_mode_within_1e12():
    level, q, T = 6, 6, 5
    src, fit, u0 = _oracle_case(level, q, verts=lattice.kuhn_tet((1, 2, 0)))
    p = DevicePlan(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows, arow=src.data, fast=True)
    us = np.stack([u0 * (t + 1) for t in range(T)])
    ub = cuda(us)
    sur = O.OracleSurrogate(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows)
    refs = us.copy()
    for _ in range(4):
        p.sweep(ub, torch.zeros_like(ub), 1)
        for t in range(T):
            O.sweeps(sur, level, src.data, refs[t], np.zeros_like(u0), 1)
        assert relerr(ub.cpu().numpy(), refs) <= 1e-12


def test_config4_slice_level7_bitwise():
    """Config 4 at full level: 33 Kuhn tets (one full group + padding group), L7, q=6 -> (4,4,5)."""
    level, q, T = 7, 6, 33
    src, fit, _ = _oracle_case(level, q, verts=lattice.kuhn_tet((0, 1, 2)))
    assert tuple(fit.degrees) == (4, 4, 5)
    mask = lattice.interior_mask(level)
    rng = np.random.default_rng(4)
    us = np.zeros((T, mask.size))
    us[:, mask] = rng.uniform(-1, 1, (T, int(mask.sum())))
    ub = cuda(us)
    p = DevicePlan(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows, arow=src.data)
    p.sweep(ub, torch.zeros_like(ub), 2)
    sur = O.OracleSurrogate(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows)
    got = ub.cpu().numpy()
    for t in (0, 17, 31, 32):
        ref = us[t].copy()
        O.sweeps(sur, level, src.data, ref, np.zeros_like(ref), 2)
        assert np.array_equal(got[t], ref), t


def test_macro_mesh_smoother_resident_equals_apply():
    from paper_2210_15280_b200 import MacroMeshSmoother
    tets = lattice.kuhn_mesh(2)          # 48 tets
    level = 4
    mm = MacroMeshSmoother(tets, level, degrees=(3, 3, 3))
    mask = lattice.interior_mask(level)
    rng = np.random.default_rng(1)
    us = np.zeros((len(tets), mask.size))
    us[:, mask] = rng.uniform(-1, 1, (len(tets), int(mask.sum())))
    u1, f = cuda(us), torch.zeros((len(tets), mask.size), dtype=torch.float64, device=DEV)
    u2 = u1.clone()
    n1 = mm.apply(u1, f, 3)
    mm.load(u2, f)
    n2 = mm.sweep(3)
    mm.store(u2)
    assert torch.equal(u1, u2)
    torch.testing.assert_close(n1, n2, rtol=1e-12, atol=0)


def test_macro_mesh_apply_host_pipelined_equals_apply():
    """End-to-end entry point (pinned host tensors, chunked two-stream pipeline) == device apply."""
    from paper_2210_15280_b200 import MacroMeshSmoother
    tets = lattice.kuhn_mesh(2)          # 48 tets
    level = 4
    mm = MacroMeshSmoother(tets, level, degrees=(3, 3, 3))
    mask = lattice.interior_mask(level)
    rng = np.random.default_rng(2)
    us = np.zeros((len(tets), mask.size))
    us[:, mask] = rng.uniform(-1, 1, (len(tets), int(mask.sum())))
    fs = np.zeros_like(us)
    fs[:, mask] = rng.standard_normal((len(tets), int(mask.sum())))
    u1, f1 = cuda(us), cuda(fs)
    n1 = mm.apply(u1, f1, 2)
    for chunk in (7, 128):
        uh = torch.from_numpy(us.copy()).pin_memory()
        fh = torch.from_numpy(fs.copy()).pin_memory()
        n2 = mm.apply_host(uh, fh, 2, chunk=chunk)
        assert torch.equal(uh, u1.cpu()), chunk
        torch.testing.assert_close(n2, n1.cpu(), rtol=1e-12, atol=0)


def test_packed_dataflow_repeatable_and_equals_simple():
    """The dataflow kernels' inter-warp / inter-CTA handoffs leave no room for races: repeated
    runs are bitwise identical and equal the one-CTA-per-tet reference-layout kernels."""
    level, q, T = 6, 5, 70
    src, fit, u0 = _oracle_case(level, q, verts=lattice.kuhn_tet((0, 2, 1)))
    rng = np.random.default_rng(9)
    us = cuda(np.stack([u0 * s for s in rng.uniform(-1, 1, T)]))
    fs = cuda(np.zeros((T, len(u0))))
    fast = DevicePlan(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows, arow=src.data)
    simple = DevicePlan(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows, arow=src.data,
                        simple=True)
    ref = us.clone()
    simple.sweep(ref, fs, 3)
    for _ in range(3):
        got = us.clone()
        fast.sweep(got, fs, 3)
        assert torch.equal(got, ref)

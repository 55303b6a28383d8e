"""Pin the C oracle against golden vectors produced by the live reference
(tests/golden/make_golden.py).  Bitwise (np.array_equal) for every kernel output;
residual norms (BLAS-order dot in the generator) to 1e-13 relative."""

import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import oracle as O

SWEEP_CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "cfg*.npz")))


def load(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def surrogate(d):
    return O.OracleSurrogate(int(d["level"]), d["lcoefs"], d["dcoefs"], str(d["variant"]), d["band_ranks"],
                             d["store_rows"])


@pytest.mark.parametrize("name", SWEEP_CASES)
def test_solve_into_matches_reference(name):
    d = load(name)
    if "solve_in" not in d:
        pytest.skip("no solve pin in this case")
    w = d["solve_in"].copy()
    surrogate(d).solve_into(w)
    assert np.array_equal(w, d["solve_out"])


@pytest.mark.parametrize("name", SWEEP_CASES)
def test_sweeps_match_reference(name):
    d = load(name)
    L, k = int(d["level"]), int(d["sweeps"])
    u = d["u0"].copy()
    norms = O.sweeps(surrogate(d), L, d["arows"], u, d["f"], 1, return_norms=True)
    assert np.array_equal(u, d["u_after_1"])
    norms = np.concatenate([norms, O.sweeps(surrogate(d), L, d["arows"], u, d["f"], k - 1, return_norms=True)])
    assert np.array_equal(u, d[f"u_after_{k}"])
    np.testing.assert_allclose(norms, d["rnorm2"], rtol=1e-13, atol=0)


@pytest.mark.parametrize("name", [n for n in SWEEP_CASES if "cfg1_L5_v1" in n or "cfg2_L4" in n])
def test_stored_ilu_matches_reference(name):
    d = load(name)
    L = int(d["level"])
    w = d["ilu_solve_in"].copy()
    O.ilu_solve_into(L, d["factors"], w)
    assert np.array_equal(w, d["ilu_solve_out"])
    u = d["u0"].copy()
    O.sweeps(None, L, d["arows"], u, d["f"], int(d["sweeps"]), factors=d["factors"])
    assert np.array_equal(u, d["ilu_u_final"])


@pytest.mark.parametrize("name", ["nddf_L3", "nddf_L4", "nddf_L5"])
@pytest.mark.parametrize("variant", ["v1", "v2"])
def test_random_coefficient_shapes(name, variant):
    """Assorted (kx+1, ky+1, kz+1) up to 9 with random tables: forward alone and full solve."""
    d = load(name)
    L = int(d["level"])
    for i, _ in enumerate(d["shapes"]):
        sur = O.OracleSurrogate(L, d[f"s{i}_lcoefs"], d[f"s{i}_dcoefs"], variant, d["band_ranks"], d[f"s{i}_store"])
        w = d[f"s{i}_w0"].copy()
        sur.forward(w)
        assert np.array_equal(w, d[f"s{i}_{variant}_fwd"])
        sur.backward(w)
        assert np.array_equal(w, d[f"s{i}_{variant}_solve"])


def test_stencil_apply_and_operator_surrogate():
    d = load("kernels_L4")
    assert np.array_equal(O.stencil_apply(4, d["arows"], d["u"]), d["stencil_out"])
    assert np.array_equal(O.stencil_apply(4, d["arow1"], d["u"]), d["stencil_out1"])
    assert np.array_equal(O.surrogate_apply_residual(4, d["acoefs"], d["u"], d["f"]), d["sres_out"])


def test_surrogate_operator_sweeps():
    d = load("sop_L4")
    u = np.zeros_like(d["f"])
    for k in (1, 2, 3):
        O.sweeps(surrogate(d), 4, None, u, d["f"], 1, acoefs=d["acoefs"])
        assert np.array_equal(u, d[f"u_after_{k}"])


def test_reference_pipeline_equivalence_recorded():
    """The stencil-form sweep the oracle restates equals Hierarchy.smooth up to CSR
    summation order (measured by make_golden.py on the live reference)."""
    m = load("meta")
    assert float(m["hierarchy_rel"]) < 1e-13
    assert bool(m["kuhn_rows_identical"])


def test_many_tets_openmp_equals_serial():
    d = load("cfg4_L4_kuhn0")
    L = int(d["level"])
    sur = surrogate(d)
    rng = np.random.default_rng(3)
    us = np.repeat(d["u0"][None], 5, axis=0) * rng.uniform(0.5, 1.5, (5, 1))
    fs = np.zeros_like(us)
    ref = us.copy()
    for t in range(5):
        O.sweeps(sur, L, d["arows"], ref[t], fs[t], 2)
    used = O.sweeps_many(sur, L, d["arows"][0], us, fs, 2, nthreads=2)
    assert used >= 1
    assert np.array_equal(us, ref)


def test_level9_oracle_run_equals_the_reference_kernels():
    """The level-9 config-3 fixture (the C oracle's 100 sweeps: what the GPU parity test and the bench's config-3
    leg are pinned to) against the REFERENCE's own Numba kernels run on the same arrays
    (tests/golden/make_l9_reference_sweeps.py): SHA-256 of the full 22.6M-entry iterate after every stored sweep."""
    import os

    import numpy as np
    import pytest

    from conftest import GOLDEN
    path = os.path.join(GOLDEN, "l9_reference_sweeps.npz")
    if not os.path.exists(path):
        pytest.skip("reference level-9 sweep fixture not generated")
    ref, ours = np.load(path), np.load(os.path.join(GOLDEN, "l9_config3.npz"))
    mine = {int(k): str(h) for k, h in zip(ours["snaps"], ours["u_sha"])}
    assert len(ref["snaps"]) >= 3
    for k, h in zip(ref["snaps"], ref["u_sha"]):
        assert mine[int(k)] == str(h), f"sweep {int(k)}"

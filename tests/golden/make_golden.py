"""Generate the golden fixtures that pin the oracle and the host setup.

Runs the UNMODIFIED reference (``/root/reference/pkg/src/tetilu``, importable in
the build container only) on small seeded cases and writes ``tests/golden/*.npz``.
The fixtures are committed; the GPU box never reads /root/reference.

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py

Every case stores its inputs (coefficients, band rows, stencil rows, seeds, vectors)
and the reference's outputs:
  * kernel pins  (P1): solve_into / stencil_apply / surrogate_apply_residual /
    CellILU outputs of the reference Numba kernels on those inputs;
  * sweep pins       : u after k smoothing steps (stencil-form cell stage,
    multigrid.py:414-429) and per-step norms;
  * setup pins   (P2): stencil_source rows, factorize_tet rows, the fitted
    surrogate arrays and effective degrees / stride of build_surrogate_ilu.
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

from tetilu import _kernels, geometry  # noqa: E402
from tetilu.assembly import CoefficientField, stencil_source  # noqa: E402
from tetilu.ilu import CellILU, factorize_tet  # noqa: E402
from tetilu.multigrid import Hierarchy, SmootherConfig  # noqa: E402
from tetilu.surrogate import build_surrogate_ilu, build_surrogate_operator  # noqa: E402

UNIT = geometry.trirect_tet(1.0)
DISTORTED = np.array([(0, 0, 0), (1, 0.1, 0), (0.2, 1, 0), (0.1, 0.3, 0.8)], dtype=float)


def kuhn_tet(path):
    p = [0, 0, 0]
    verts = [tuple(p)]
    for axis in path:
        p[axis] = 1
        verts.append(tuple(p))
    return np.array(verts, dtype=float)


def diag_tensor(d):
    d = np.asarray(d, dtype=float)
    return CoefficientField.tensor(lambda pts: np.broadcast_to(np.diag(d), (len(np.atleast_2d(pts)), 3, 3)))


def sinkappa():
    def fn(p):
        p = np.atleast_2d(p)
        return 1.0 + 0.5 * np.sin(2 * np.pi * p[:, 0]) * np.sin(2 * np.pi * p[:, 1]) * np.sin(2 * np.pi * p[:, 2])
    return CoefficientField.scalar(fn, name="sinkappa")


def interior_mask(level):
    return geometry.is_interior(geometry.enumerate_grid(level), level)


def ref_sweep(sur, src, u, f):
    """One stencil-form cell stage: r = A u, w = f - r (interior), solve, u += w."""
    level = src.level
    n = 2 ** level
    _, rowoff = geometry.rank_tables(level)
    arows, aconst = src.kernel_args
    mask = interior_mask(level)
    r = np.zeros_like(u)
    _kernels.stencil_apply(n, rowoff, arows, aconst, u, r)
    w = np.zeros_like(u)
    w[mask] = f[mask] - r[mask]
    rn2 = float(np.dot(w, w))  # ||f - A u||^2 before the solve (BLAS order; compare with rtol)
    sur.solve_into(w)
    u[mask] += w[mask]
    return rn2


def surrogate_arrays(prefix, sur):
    return {
        f"{prefix}lcoefs": sur._lcoefs, f"{prefix}dcoefs": sur._dcoefs,
        f"{prefix}band_ranks": sur._band_ranks, f"{prefix}store_rows": sur._store_rows,
        f"{prefix}eff_degrees": np.array(sur.degrees, dtype=np.int64),
        f"{prefix}stride": np.array(sur.stride), f"{prefix}variant": np.array(sur.variant),
    }


def case_sweeps(name, verts, coeff, level, q, variant, sweeps, seed, f_kind="zero",
                u_kind="uniform", store_src=True, stored_ilu=False, solve_seed=None):
    tet = geometry.MacroTet(verts)
    src = stencil_source(tet, level, coeff)
    sur = build_surrogate_ilu(src, level, (q, q, q), variant=variant)
    grid = geometry.grid_size(level)
    mask = interior_mask(level)
    rng = np.random.default_rng(seed)
    nint = int(mask.sum())
    u0 = np.zeros(grid)
    f = np.zeros(grid)
    if u_kind == "uniform":
        u0[mask] = rng.uniform(-1.0, 1.0, nint)
    if f_kind == "normal":
        f[mask] = rng.standard_normal(nint)
    u = u0.copy()
    unorms, rnorm2, snaps = [], [], {}
    for k in range(sweeps):
        rnorm2.append(ref_sweep(sur, src, u, f))
        unorms.append(float(np.linalg.norm(u)))
        if k in (0, 1, sweeps - 1):
            snaps[k + 1] = u.copy()
    d = {"level": np.array(level), "q": np.array(q), "sweeps": np.array(sweeps),
         "u0": u0, "f": f, "unorms": np.array(unorms), "rnorm2": np.array(rnorm2),
         "src_constant": np.array(src.constant), "verts": np.asarray(verts, float)}
    for k, v in snaps.items():
        d[f"u_after_{k}"] = v
    d.update(surrogate_arrays("", sur))
    d["arows"] = np.atleast_2d(src.data) if (store_src or src.constant) else np.atleast_2d(src.data[0])
    if solve_seed is not None:
        w = np.zeros(grid)
        w[mask] = np.random.default_rng(solve_seed).standard_normal(nint)
        d["solve_in"] = w.copy()
        sur.solve_into(w)
        d["solve_out"] = w
    if stored_ilu:
        res = factorize_tet(src, level)
        cell = CellILU(res)
        d["factors"] = res.rows
        u = u0.copy()
        for _ in range(sweeps):
            ref_sweep(cell, src, u, f)
        d["ilu_u_final"] = u
        w = np.zeros(grid)
        w[mask] = np.random.default_rng(seed + 100).standard_normal(nint)
        d["ilu_solve_in"] = w.copy()
        cell.solve_into(w)
        d["ilu_solve_out"] = w
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **d)
    print(f"{name}: eff={sur.degrees} stride={sur.stride} band={len(sur._band_ranks)} "
          f"rho_last={unorms[-1] / unorms[-2] if sweeps > 1 and unorms[-2] else float('nan'):.6f}")
    return src, sur


def case_random_nddf(name, level, shapes, seed):
    """Random coefficient tables of assorted degree shapes -> fwd / full solve outputs."""
    rng = np.random.default_rng(seed)
    n = 2 ** level
    _, rowoff = geometry.rank_tables(level)
    grid = geometry.grid_size(level)
    mask = interior_mask(level)
    band = geometry.lattice_rank(geometry.enumerate_grid(level, "interior"), level)
    coords = geometry.enumerate_grid(level, "interior")
    bmask = (coords == 1).any(axis=1) | (coords.sum(axis=1) == n - 1)
    band = band[bmask]
    d = {"level": np.array(level), "band_ranks": band}
    for i, (kx1, ky1, kz1) in enumerate(shapes):
        lco = rng.standard_normal((7, kx1, ky1, kz1)) * 0.05
        dco = 1.0 + 0.1 * rng.standard_normal((1, kx1, ky1, kz1))
        store = rng.standard_normal((len(band), 9)) * 0.05
        store[:, 8] = 1.0 + 0.1 * rng.random(len(band))
        w0 = np.zeros(grid)
        w0[mask] = rng.standard_normal(int(mask.sum()))
        d[f"s{i}_lcoefs"], d[f"s{i}_dcoefs"], d[f"s{i}_store"], d[f"s{i}_w0"] = lco, dco, store, w0
        for variant in ("v1", "v2"):
            use = variant == "v1"
            w = w0.copy()
            _kernels.surrogate_forward(n, rowoff, 1.0 / n, lco, w, use, band, store)
            d[f"s{i}_{variant}_fwd"] = w.copy()
            _kernels.surrogate_backward(n, rowoff, 1.0 / n, lco, dco, w, use, band, store)
            d[f"s{i}_{variant}_solve"] = w
    d["shapes"] = np.array(shapes, dtype=np.int64)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **d)
    print(f"{name}: shapes={shapes}")


def case_kernels_misc(name, level, seed):
    """stencil_apply with per-point rows and surrogate_apply_residual on random inputs."""
    rng = np.random.default_rng(seed)
    n = 2 ** level
    _, rowoff = geometry.rank_tables(level)
    grid = geometry.grid_size(level)
    mask = interior_mask(level)
    u = np.zeros(grid)
    f = np.zeros(grid)
    u[mask] = rng.standard_normal(int(mask.sum()))
    f[mask] = rng.standard_normal(int(mask.sum()))
    arows = rng.standard_normal((grid, 15))
    out = np.zeros(grid)
    _kernels.stencil_apply(n, rowoff, arows, False, u, out)
    arow1 = rng.standard_normal((1, 15))
    out1 = np.zeros(grid)
    _kernels.stencil_apply(n, rowoff, arow1, True, u, out1)
    acoefs = rng.standard_normal((15, 4, 3, 2))
    wres = np.zeros(grid)
    _kernels.surrogate_apply_residual(n, rowoff, 1.0 / n, acoefs, u, f, wres)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), level=np.array(level), u=u, f=f,
                        arows=arows, stencil_out=out, arow1=arow1, stencil_out1=out1,
                        acoefs=acoefs, sres_out=wres)
    print(f"{name}: ok")


def case_surrogate_operator(name, level, q, aq, seed):
    """a_mode='surrogate' sweeps (SurrogateOperator.residual_into, surrogate.py:344-358)."""
    tet = geometry.MacroTet(UNIT)
    src = stencil_source(tet, level, sinkappa())
    sur = build_surrogate_ilu(src, level, (q, q, q), variant="v1")
    op = build_surrogate_operator(src, level, (aq, aq, aq))
    grid = geometry.grid_size(level)
    mask = interior_mask(level)
    rng = np.random.default_rng(seed)
    u = np.zeros(grid)
    f = np.zeros(grid)
    f[mask] = rng.standard_normal(int(mask.sum()))
    out = {}
    for k in range(3):
        w = np.zeros(grid)
        op.residual_into(u, f, w)
        sur.solve_into(w)
        u[mask] += w[mask]
        out[f"u_after_{k + 1}"] = u.copy()
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), level=np.array(level), f=f,
                        acoefs=op._acoefs, **surrogate_arrays("", sur), **out)
    print(f"{name}: a-degrees={op._acoefs.shape[1:]}")


def check_hierarchy_equivalence(level=4, q=4):
    """The stencil-form pipeline equals Hierarchy.smooth up to CSR summation order."""
    mesh = geometry.single_tet_mesh(UNIT)
    hier = Hierarchy(mesh, 2, level, smoother=SmootherConfig("surrogate_ilu", (q, q, q)))
    sp = hier.space(hier.top)
    rng = np.random.default_rng(7)
    u = np.where(sp.free, rng.uniform(-1, 1, sp.ndof), 0.0)
    f = np.zeros(sp.ndof)
    u2 = u.copy()
    hier.smooth(hier.top, u, f)
    src = hier.sources[hier.top][0]
    sur = hier.cell_preconditioners(hier.top)[0]
    ref_sweep(sur, src, u2, f)
    rel = float(np.abs(u - u2).max() / np.abs(u).max())
    print(f"Hierarchy.smooth vs stencil pipeline (L{level}): max rel diff {rel:.3e}")
    return rel


def main():
    cases = {}
    # configs[0]: unit tet, Poisson, q=4 (eff (4,4,4) at L5), 20 sweeps; V1, V2, stored ILU
    case_sweeps("cfg1_L5_v1", UNIT, CoefficientField.constant(1.0), 5, 4, "v1", 20, 1,
                stored_ilu=True, solve_seed=11)
    case_sweeps("cfg1_L5_v2", UNIT, CoefficientField.constant(1.0), 5, 4, "v2", 20, 1, solve_seed=11)
    # configs[1] geometry/coefficient at a CPU-friendly level (per-point tensor rows)
    case_sweeps("cfg2_L4_v1", DISTORTED, diag_tensor((1, 1, 1e-3)), 4, 6, "v1", 10, 2,
                stored_ilu=True, solve_seed=12)
    case_sweeps("cfg2_L5_v1", DISTORTED, diag_tensor((1, 1, 1e-3)), 5, 6, "v1", 5, 2, solve_seed=12)
    # configs[4]: degree sweep q=0..8 at L4 (distorted tet, K=diag(1,1e-2,1))
    for q in range(0, 9):
        case_sweeps(f"cfg5_L4_q{q}", DISTORTED, diag_tensor((1, 1e-2, 1)), 4, q, "v1", 6, 5,
                    solve_seed=15)
    case_sweeps("cfg5_L5_q2_v2", DISTORTED, diag_tensor((1, 1e-2, 1)), 5, 2, "v2", 4, 5, solve_seed=15)
    # configs[2] coefficient k = 1 + 0.5 sin sin sin; f ~ N(0,1), u = 0
    case_sweeps("cfg3_L4_v1", UNIT, sinkappa(), 4, 6, "v1", 3, 3, f_kind="normal", u_kind="zero",
                solve_seed=13)
    case_sweeps("cfg3_L5_v1", UNIT, sinkappa(), 5, 6, "v1", 3, 3, f_kind="normal", u_kind="zero")
    # configs[3]: Kuhn tets of a unit cube (all 6 vertex paths), Poisson, q=6
    from itertools import permutations
    rows = []
    for i, path in enumerate(permutations(range(3))):
        src, _ = case_sweeps(f"cfg4_L4_kuhn{i}", kuhn_tet(path), CoefficientField.constant(1.0), 4, 6,
                             "v1", 4, 4, solve_seed=14)
        rows.append(src.data)
    cases["kuhn_rows_identical"] = all(np.array_equal(rows[0], r) for r in rows)
    print("kuhn stencils identical:", cases["kuhn_rows_identical"])
    case_sweeps("cfg4_L5_kuhn0", kuhn_tet((0, 1, 2)), CoefficientField.constant(1.0), 5, 6, "v1", 3, 4)
    # kernel-level pins on random inputs
    case_random_nddf("nddf_L4", 4, [(1, 1, 1), (3, 2, 4), (5, 5, 6), (2, 5, 1)], 21)
    case_random_nddf("nddf_L5", 5, [(5, 5, 5), (9, 9, 9), (4, 1, 3)], 22)
    case_random_nddf("nddf_L3", 3, [(5, 5, 6), (1, 2, 1)], 23)
    case_kernels_misc("kernels_L4", 4, 31)
    case_surrogate_operator("sop_L4", 4, 4, 3, 41)
    rel = check_hierarchy_equivalence()
    np.savez_compressed(os.path.join(OUT, "meta.npz"), hierarchy_rel=np.array(rel),
                        kuhn_rows_identical=np.array(cases["kuhn_rows_identical"]),
                        numpy_version=np.array(np.__version__))


if __name__ == "__main__":
    main()

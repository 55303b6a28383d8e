"""Locate plane-path mismatches vs the oracle (debug tool).  TILU_PLANE_DEBUG=1: forward pass only."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from oracle import oracle as O
from paper_2210_15280_b200 import DevicePlan, lattice, fitting as F, stencil as S

fwd_only = os.environ.get("TILU_PLANE_DEBUG") == "1"
for (level, q, variant, fseed) in [(6, 0, "v2", None), (6, 3, "v1", 6), (7, 4, "v2", None)]:
    src = S.stencil_source(lattice.unit_tet(), level, S.CoefficientField.constant(1.0))
    fit = F.fit_surrogate_ilu(src, level, (q, q, q), variant)
    mask = lattice.interior_mask(level)
    u0 = np.zeros(lattice.grid_size(level)); u0[mask] = np.random.default_rng(0).uniform(-1, 1, int(mask.sum()))
    f = np.zeros_like(u0)
    if fseed is not None:
        f[mask] = np.random.default_rng(fseed).normal(size=int(mask.sum()))
    sur = O.OracleSurrogate(level, fit.lcoefs, fit.dcoefs, variant, fit.band_ranks, fit.store_rows)
    if fwd_only:
        ref = np.zeros_like(u0)
        ref[mask] = (f - O.stencil_apply(level, src.data, u0))[mask]
        sur.forward(ref)
    else:
        ref = u0.copy()
        O.sweeps(sur, level, src.data, ref, f, 1)
    p = DevicePlan(level, fit.lcoefs, fit.dcoefs, variant, fit.band_ranks, fit.store_rows, arow=src.data, schedule="plane")
    u = torch.as_tensor(u0, device="cuda")
    p.sweep(u, torch.as_tensor(f, device="cuda"), 1)
    got = u.cpu().numpy()
    bad = np.nonzero((got != ref) & mask)[0]
    print(f"{'FWD ' if fwd_only else ''}L{level} q{q} {variant}: {len(bad)} of {int(mask.sum())} differ; max rel {np.abs(got-ref).max()/np.abs(ref).max():.3e}", flush=True)
    if len(bad):
        xyz = lattice.lattice_coords(level, 'full')[bad]
        s = xyz[:, 1] + xyz[:, 2]
        print("  z range", xyz[:, 2].min(), xyz[:, 2].max(), " s range", s.min(), s.max(), " x range", xyz[:, 0].min(), xyz[:, 0].max())
        t = xyz[:, 0] + 2 * xyz[:, 1] + 3 * xyz[:, 2]
        order = np.argsort(t, kind="stable")
        print("  smallest t:", [tuple(int(a) for a in v) for v in xyz[order[:10]]])
        order = np.argsort(-t, kind="stable")
        print("  largest t:", [tuple(int(a) for a in v) for v in xyz[order[:10]]])
        print("  by chunk:", np.bincount(xyz[:, 2] // 32).tolist(), " by band:", np.bincount((s - 2) // 4).tolist()[:40])
        e = np.abs(got - ref)[bad]
        worst = np.argsort(-e)[:5]
        print("  worst:", [(tuple(int(a) for a in xyz[i]), float(e[i])) for i in worst])

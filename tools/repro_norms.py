"""Repro of test_batched_tets_equal_single[False] with launch blocking and per-call checks."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2210_15280_b200 import DevicePlan, _lib, fitting, lattice, stencil  # noqa: E402

level, q, T = 5, 6, int(os.environ.get("T", "7"))
src = stencil.stencil_source(lattice.kuhn_tet((0, 1, 2)), level, stencil.CoefficientField.constant(1.0))
fit = fitting.fit_surrogate_ilu(src, level, (q, q, q), "v1")
mask = lattice.interior_mask(level)
u0 = np.zeros(mask.size)
u0[mask] = np.random.default_rng(0).uniform(-1, 1, int(mask.sum()))
us = np.stack([u0 * s for s in np.random.default_rng(5).uniform(0.5, 2.0, T)])
fs = np.zeros_like(us)
fs[2 % T] = u0
p = DevicePlan(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows, arow=src.data)
for trial in range(int(os.environ.get("TRIALS", "5"))):
    ub = torch.as_tensor(us, device="cuda")
    norms = os.environ.get("NORMS", "1") == "1"
    rn = p.sweep(ub, torch.as_tensor(fs, device="cuda"), int(os.environ.get("SWEEPS", "2")), norms=norms)
    torch.cuda.synchronize()
    print("trial", trial, "ok", float(ub.abs().sum()), flush=True)

"""Tiny batched-path run (level 4, 7 tets) for compute-sanitizer."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2210_15280_b200 import DevicePlan, fitting, lattice, stencil  # noqa: E402

level = int(os.environ.get("LEVEL", "4"))
T = int(os.environ.get("T", "7"))
src = stencil.stencil_source(lattice.kuhn_tet((0, 1, 2)), level, stencil.CoefficientField.constant(1.0))
q = int(os.environ.get("Q", "3"))
fit = fitting.fit_surrogate_ilu(src, level, (q, q, q), "v1")
p = DevicePlan(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows, arow=src.data)
mask = lattice.interior_mask(level)
u = np.zeros((T, mask.size))
u[:, mask] = np.random.default_rng(0).uniform(-1, 1, (T, int(mask.sum())))
ut = torch.as_tensor(u, device="cuda")
p.sweep(ut, torch.zeros_like(ut), 1)
torch.cuda.synchronize()
print("ok", float(ut.abs().sum()))

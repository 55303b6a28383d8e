"""Profiling driver: config-4 workload (384 Kuhn tets, L7, q=6) on the resident packed path.
Used under ncu (one GPU):  ncu ... python tools/prof_batch.py [--tets N] [--sweeps S] [--fast]"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("--tets", type=int, default=384)
ap.add_argument("--level", type=int, default=7)
ap.add_argument("--sweeps", type=int, default=2)
ap.add_argument("--fast", action="store_true")
a = ap.parse_args()

import torch  # noqa: E402

from paper_2210_15280_b200 import DevicePlan, fitting, lattice, stencil  # noqa: E402

src = stencil.stencil_source(lattice.kuhn_tet((0, 1, 2)), a.level, stencil.CoefficientField.constant(1.0))
fit = fitting.fit_surrogate_ilu(src, a.level, (6, 6, 6), "v1")
p = DevicePlan(a.level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows, arow=src.data, fast=a.fast)
mask = lattice.interior_mask(a.level)
u = torch.zeros((a.tets, mask.size), dtype=torch.float64, device="cuda")
u[:, torch.as_tensor(mask, device="cuda")] = torch.rand((a.tets, int(mask.sum())), dtype=torch.float64,
                                                        device="cuda") * 2 - 1
up = p.pack(u)
fp = p.pack(torch.zeros_like(u))
wp = p.new_scratch(a.tets)
for _ in range(a.sweeps):
    p.sweep_packed(up, fp, wp, a.tets, 1, norms=True)
torch.cuda.synchronize()
print("ok", float(up.abs().sum()))

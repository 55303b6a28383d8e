"""Sweep time of the batched kernels vs the number of macro-tets on one GPU (the per-rank share of config 4 at
1, 2, 4, 8 GPUs: 384 / 192 / 96 / 48 tets), level 7, q = 6, resident packed state.  TILU_TPL=1|2 overrides the
tets-per-lane choice.   python tools/tets_scan.py [--tets 48 96 192 384]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_15280_b200 import DevicePlan, _lib, fitting, lattice, stencil  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tets", type=int, nargs="*", default=[48, 96, 192, 384])
ap.add_argument("--level", type=int, default=7)
ap.add_argument("--sweeps", type=int, default=20)
a = ap.parse_args()
src = stencil.stencil_source(lattice.kuhn_tet((0, 1, 2)), a.level, stencil.CoefficientField.constant(1.0))
fit = fitting.fit_surrogate_ilu(src, a.level, (6, 6, 6), "v1", factorize="device")
p = DevicePlan(a.level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows, arow=src.data)
mask = torch.as_tensor(lattice.interior_mask(a.level), device="cuda")
N = int(mask.sum())
for nt in a.tets:
    u = torch.zeros((nt, mask.numel()), dtype=torch.float64, device="cuda")
    u[:, mask] = torch.rand((nt, N), dtype=torch.float64, device="cuda") * 2 - 1
    up, fp, wp = p.pack(u), p.pack(torch.zeros_like(u)), p.new_scratch(nt)
    p.sweep_packed(up, fp, wp, nt, 3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    p.sweep_packed(up, fp, wp, nt, a.sweeps)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.sweeps
    print(json.dumps({"tets": nt, "tpl_env": os.environ.get("TILU_TPL"), "ms_per_sweep": ms,
                      "dof_updates_per_s": nt * N / (ms * 1e-3)}), flush=True)

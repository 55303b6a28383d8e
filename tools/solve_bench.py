"""Time the drop-in SurrogateILU.solve_into (tilu_solve_into) per level: the sweep-routed fast kernels
(default) vs the reference-layout kernels (schedule='simple'), and check them against each other bitwise."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_15280_b200 import DevicePlan, fitting, lattice, stencil  # noqa: E402

out = []
for level, ntets in ((5, 1), (6, 1), (7, 1), (8, 1), (7, 48)):
    src = stencil.stencil_source(lattice.unit_tet(), level, stencil.CoefficientField.constant(1.0))
    fit = fitting.fit_surrogate_ilu(src, level, (4, 4, 4), "v1", factorize="device")
    base = (level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows)
    mask = torch.as_tensor(lattice.interior_mask(level), device="cuda")
    w0 = torch.zeros((ntets, mask.numel()), dtype=torch.float64, device="cuda")
    w0[:, mask] = torch.randn((ntets, int(mask.sum())), dtype=torch.float64, device="cuda")
    res = {}
    for sched in ("auto", "simple"):
        p = DevicePlan(*base, schedule=sched)          # no operator: the pure preconditioner (SurrogateILU.plan())
        w = w0.clone()
        p.solve_into(w)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        ws = [w0.clone() for _ in range(reps)]
        a.record()
        for x in ws:
            p.solve_into(x)
        b.record()
        torch.cuda.synchronize()
        res[sched] = (a.elapsed_time(b) / reps, w)
    rec = {"level": level, "ntets": ntets, "ms_fast": res["auto"][0], "ms_reference_layout": res["simple"][0],
           "bitwise_equal": bool(torch.equal(res["auto"][1], res["simple"][1]))}
    out.append(rec)
    print(json.dumps(rec), flush=True)

"""Time one sweep of a single macro-tet (constant coefficient, unit tet) at a given level through
the batched kernels (1 tet in a 32-lane group) and, for small levels, the reference-layout kernels."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2210_15280_b200 import DevicePlan, _lib, fitting, lattice, stencil  # noqa: E402

level = int(os.environ.get("LEVEL", "9"))
q = int(os.environ.get("Q", "6"))
t0 = time.time()
src = stencil.stencil_source(lattice.unit_tet(), level, stencil.CoefficientField.constant(1.0))
fit = fitting.fit_surrogate_ilu(src, level, (q, q, q), "v1")
print(f"setup L{level}: {time.time() - t0:.1f}s eff {fit.degrees}", flush=True)
p = DevicePlan(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows, arow=src.data)
N = lattice.interior_size(level)
up = torch.rand(p.packed_numel(1), dtype=torch.float64, device="cuda")
fp = torch.zeros_like(up)
wp = p.new_scratch(1)
for _ in range(2):
    p.sweep_packed(up, fp, wp, 1, 1)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    p.sweep_packed(up, fp, wp, 1, 1)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
print(f"batched kernels, 1 tet L{level}: {ms:.2f} ms/sweep = {N / (ms * 1e-3):.3e} DoF-upd/s", flush=True)

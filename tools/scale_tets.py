"""Time one packed sweep vs. the number of tets (critical-path vs throughput diagnosis)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2210_15280_b200 import DevicePlan, _lib, fitting, lattice, stencil  # noqa: E402

level = int(os.environ.get("LEVEL", "7"))
src = stencil.stencil_source(lattice.kuhn_tet((0, 1, 2)), level, stencil.CoefficientField.constant(1.0))
fit = fitting.fit_surrogate_ilu(src, level, (6, 6, 6), "v1")
p = DevicePlan(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows, arow=src.data)
grid = lattice.grid_size(level)
for T in [int(t) for t in os.environ.get("TETS", "32,64,128,256,384,768").split(",")]:
    up = torch.rand(p.packed_numel(T), dtype=torch.float64, device="cuda")
    fp = torch.zeros_like(up)
    wp = p.new_scratch(T)
    for _ in range(2):
        p.sweep_packed(up, fp, wp, T, 1)
    _lib.profile_enable(True)
    for _ in range(3):
        p.sweep_packed(up, fp, wp, T, 1)
    torch.cuda.synchronize()
    prof = _lib.profile_read()
    _lib.profile_enable(False)
    f, b = prof["batch_fwd"], prof["batch_bwd"]
    print(f"tets {T:4d}  fwd {f[1]/f[0]:.3f} ms  bwd {b[1]/b[0]:.3f} ms  "
          f"rate {T * lattice.interior_size(level) / ((f[1]/f[0] + b[1]/b[0]) * 1e-3):.3e} DoF-upd/s", flush=True)

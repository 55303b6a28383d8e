"""Sentinel statistics of one packed sweep (needs a -DTILU_STATS build: TILU_LIB=.../libtilu_stats.so)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2210_15280_b200 import DevicePlan, _lib, fitting, lattice, stencil  # noqa: E402

level = int(os.environ.get("LEVEL", "7"))
src = stencil.stencil_source(lattice.kuhn_tet((0, 1, 2)), level, stencil.CoefficientField.constant(1.0))
fit = fitting.fit_surrogate_ilu(src, level, (6, 6, 6), "v1")
p = DevicePlan(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows, arow=src.data)
L = _lib.lib()
st = (ctypes.c_ulonglong * 4)()
for T in [int(t) for t in os.environ.get("TETS", "32,384").split(",")]:
    up = torch.rand(p.packed_numel(T), dtype=torch.float64, device="cuda")
    fp = torch.zeros_like(up)
    wp = p.new_scratch(T)
    p.sweep_packed(up, fp, wp, T, 1)
    torch.cuda.synchronize()
    L.tilu_stats_read(st)
    p.sweep_packed(up, fp, wp, T, 1)
    torch.cuda.synchronize()
    L.tilu_stats_read(st)
    print(f"tets {T}: warp-points {st[0]}  with sentinel {st[1]} ({100 * st[1] / max(st[0], 1):.1f}%)  "
          f"re-reads {st[2]} ({st[2] / max(st[0], 1):.3f}/point)", flush=True)

"""Time the single-tet sweep (plane kernels vs interleaved kernels) on one macro-tet.

    LEVEL=9 Q=6 FAST=0 SWEEPS=10 COEF=sin python tools/plane_bench.py

Unit tet, V1, u ~ U[-1, 1], f ~ N(0, 1); COEF=sin: config 3's k(x) with the rows evaluated on the
fly (separable tables), COEF=one: constant coefficient.
Prints ms/sweep and DoF-updates/s of tilu_sweep (pack + sweeps + unpack inside) and the per-kernel
device times from the library's event profiler.
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2210_15280_b200 import DevicePlan, _lib, fitting, lattice, stencil  # noqa: E402

level = int(os.environ.get("LEVEL", "9"))
q = int(os.environ.get("Q", "6"))
fast = os.environ.get("FAST", "0") == "1"
sweeps = int(os.environ.get("SWEEPS", "10"))
scheds = os.environ.get("SCHED", "plane").split(",")
variant = os.environ.get("VARIANT", "v1")
t0 = time.time()
coef = os.environ.get("COEF", "sin")
src = stencil.stencil_source(lattice.unit_tet(), level,
                             stencil.sin_kappa() if coef == "sin" else stencil.CoefficientField.constant(1.0))
op = {"sepk": src.sepk} if src.sepk is not None else {"arow": src.data}
fit = fitting.fit_surrogate_ilu(src, level, (q, q, q), variant)
print(f"setup L{level}: {time.time() - t0:.1f}s eff {fit.degrees}", flush=True)
N = lattice.interior_size(level)
mask = lattice.interior_mask(level)
rng = np.random.default_rng(3)
u0 = np.zeros(lattice.grid_size(level))
u0[mask] = rng.uniform(-1, 1, int(mask.sum()))
f0 = np.zeros_like(u0)
f0[mask] = rng.normal(size=int(mask.sum()))
for sched in scheds:
    p = DevicePlan(level, fit.lcoefs, fit.dcoefs, variant, fit.band_ranks, fit.store_rows, fast=fast, schedule=sched,
                   **op)
    u = torch.as_tensor(u0, device="cuda")
    f = torch.as_tensor(f0, device="cuda")
    p.sweep(u, f, 2)
    torch.cuda.synchronize()
    _lib.profile_enable(True)
    _lib.profile_read()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rn = p.sweep(u, f, sweeps, norms=True)
    e1.record()
    torch.cuda.synchronize()
    prof = _lib.profile_read()
    _lib.profile_enable(False)
    ms = e0.elapsed_time(e1) / sweeps
    print(f"[{sched}{' fast' if fast else ''}] L{level}: {ms:.3f} ms/sweep = {N / (ms * 1e-3):.3e} DoF-upd/s; "
          f"rnorm2 first/last {rn[0].item():.6e} {rn[-1].item():.6e}", flush=True)
    for k, (cnt, tms) in sorted(prof.items()):
        print(f"    {k:16s} {cnt:5d} launches {tms / max(cnt, 1):9.4f} ms avg", flush=True)

"""Small invocations of every kernel family, for the bounds-checked build (compute-sanitizer is not
available on the GPU pool):
    python tools/build_variant.py bounds -DTILU_DEBUG_BOUNDS
    TILU_LIB=paper_2210_15280_b200/lib/variants/libtilu_bounds.so python tools/small_cases.py
reference-layout (simple) kernels, plane-layout band kernels (const row, per-point rows, on-the-fly
separable rows, stored factors), batched dataflow kernels (1 and 2 tets per lane), residual /
stencil apply / operator surrogate, levels 3-5."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2210_15280_b200 import DevicePlan, fitting, lattice, stencil  # noqa: E402


def u0(level, t=1):
    m = lattice.interior_mask(level)
    u = np.zeros((t, m.size))
    u[:, m] = np.random.default_rng(0).uniform(-1, 1, (t, int(m.sum())))
    return torch.as_tensor(u if t > 1 else u[0], device="cuda")


for level in (3, 4, 5):
    src = stencil.stencil_source(lattice.unit_tet(), level, stencil.sin_kappa())
    fit = fitting.fit_surrogate_ilu(src, level, (3, 3, 3), "v1")
    base = (level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows)
    for sched in ("simple", "plane"):
        for op in ({"sepk": src.sepk}, {"arows": src.data}):
            p = DevicePlan(*base, schedule=sched, **op)
            u = u0(level)
            p.sweep(u, torch.zeros_like(u), 2, norms=True)
            p.residual(u, torch.zeros_like(u), norms=True)
            p.solve_into(u)
    one = stencil.stencil_source(lattice.kuhn_tet((0, 1, 2)), level, stencil.CoefficientField.constant(1.0))
    fk = fitting.fit_surrogate_ilu(one, level, (3, 3, 3), "v1")
    for T in (2, 40):
        p = DevicePlan(level, fk.lcoefs, fk.dcoefs, "v1", fk.band_ranks, fk.store_rows, arow=one.data)
        u = u0(level, T)
        p.sweep(u, torch.zeros_like(u), 2, norms=True)
    fr = fitting.factorize_tet(src, level, full_store=True)
    p = DevicePlan(level, np.zeros((7, 1, 1, 1)), np.zeros(1), "v2", factors=fr.rows, sepk=src.sepk, schedule="plane")
    u = u0(level)
    p.sweep(u, torch.zeros_like(u), 2, stored=True)
    ac = fitting.fit_surrogate_operator(src, level, (2, 2, 2))
    p = DevicePlan(*base, acoefs=ac)
    u = u0(level)
    p.sweep(u, torch.zeros_like(u), 2, norms=True)
    torch.cuda.synchronize()
    print(f"level {level} ok", flush=True)
print("sanitize cases done")

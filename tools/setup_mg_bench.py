"""Measure the 8(f) rows on the GPU: on-device factorization vs the host routine (levels 7-9, constant
and on-the-fly separable rows) and the multigrid V-cycle around the smoother (convergence factor and
time per cycle).  Prints one JSON object; `python tools/setup_mg_bench.py [--levels 7 8 9] [--mg 7]`."""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_15280_b200 import SmootherConfig, lattice  # noqa: E402
from paper_2210_15280_b200 import fitting as F  # noqa: E402
from paper_2210_15280_b200 import multigrid as MG  # noqa: E402
from paper_2210_15280_b200 import stencil as S  # noqa: E402


def time_factor(level, kind, reps=3):
    if kind == "const":
        src = S.stencil_source(lattice.unit_tet(), level, S.CoefficientField.constant(1.0))
    else:
        coeff = S.sin_kappa()
        sk = S.SeparableK(level, coeff.tables(level), coeff.c0, S.separable_program(lattice.unit_tet(), level)[1])
        src = S.StencilSource(level, None, False, sk)       # device path: no [grid, 15] rows at all
    band = lattice.band_ranks(level)
    F.factorize_tet_device(src, level, full_store=False, collect_ranks=band)  # warm-up
    torch.cuda.synchronize()
    td = []
    for _ in range(reps):
        t = time.perf_counter()
        dev = F.factorize_tet_device(src, level, full_store=False, collect_ranks=band)
        torch.cuda.synchronize()
        td.append(time.perf_counter() - t)
    from paper_2210_15280_b200 import _lib
    _lib.profile_enable(True)
    F.factorize_tet_device(src, level, full_store=False, collect_ranks=band)
    torch.cuda.synchronize()
    prof = _lib.profile_read()
    _lib.profile_enable(False)
    kms = prof["factorize"][1] / prof["factorize"][0]
    n_int = lattice.interior_size(level)
    out = {"level": level, "rows": kind, "interior": n_int, "wavefronts": 3 * 2 ** level - 11,
           "device_s": min(td), "device_points_per_s": n_int / min(td),
           "kernel_ms": kms, "kernel_us_per_wavefront": 1e3 * kms / (3 * 2 ** level - 11),
           # algorithmic bytes: the 72-byte factor row written per point (+ 120 B of per-point operator rows when
           # they are read; constant / on-the-fly rows read nothing)
           "kernel_algorithmic_gbs": n_int * 72 / (kms * 1e-3) / 1e9}
    if kind == "const" or level <= 8:
        hsrc = src if kind == "const" else S.stencil_source(lattice.unit_tet(), level, S.sin_kappa())
        t = time.perf_counter()
        host = F.factorize_tet(hsrc, level, full_store=False, collect_ranks=band)
        out["host_s"] = time.perf_counter() - t
        out["bitwise_equal"] = bool(np.array_equal(host.collected, dev.collected))
        out["speedup"] = out["host_s"] / out["device_s"]
    return out


def time_mg(lmax, nu=2, steps=8):
    t = time.perf_counter()
    H = MG.Hierarchy(lattice.unit_tet(), 2, lmax, S.CoefficientField.constant(1.0),
                     SmootherConfig(kind="surrogate_ilu", degrees=(3, 3, 3)), nu, nu, factorize="device")
    setup = time.perf_counter() - t
    rho = H.convergence_factor(steps=steps)
    g = lattice.grid_size(lmax)
    f = torch.as_tensor(np.where(lattice.interior_mask(lmax), np.random.default_rng(1).standard_normal(g), 0.0), device="cuda")
    u = H.zero(H.top)
    H.v_cycle(H.top, u, f)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        H.v_cycle(H.top, u, f)
    b.record()
    torch.cuda.synchronize()
    u2, cycles = H.solve(f, tol=1e-10)
    return {"lmax": lmax, "lmin": 2, "nu_pre": nu, "nu_post": nu, "setup_s": setup, "rho": rho, "rho_steps": steps,
            "ms_per_v_cycle": a.elapsed_time(b) / 5, "interior": lattice.interior_size(lmax),
            "solve_cycles_to_1e-10": cycles}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--levels", type=int, nargs="*", default=[7, 8, 9])
    ap.add_argument("--mg", type=int, nargs="*", default=[6, 7])
    a = ap.parse_args()
    res = {"factorize": [], "multigrid": []}
    for L in a.levels:
        for kind in ("const", "sepk"):
            res["factorize"].append(time_factor(L, kind))
            print(json.dumps(res["factorize"][-1]), flush=True)
    for L in a.mg:
        res["multigrid"].append(time_mg(L))
        print(json.dumps(res["multigrid"][-1]), flush=True)
    print(json.dumps(res))

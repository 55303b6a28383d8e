"""Per-configuration measurements beyond the bench line (BASELINE.json configs 1, 2, 5):
GPU throughput of the single-tet path, the convergence rate next to the C oracle's (3 significant
digits required), and for configs 1 and 5 the stored-factor ILU(0) sweep (CellILU) per degree.

    python tools/configs_bench.py [--configs 1,2,5] [--level5 8] > profiles/<tag>_configs.json

Inputs are synthetic per BASELINE.json: u ~ U[-1, 1] (seed = config number), f = 0, Dirichlet 0.
The rate is the reference's last-step ratio ||u_k|| / ||u_{k-1}|| (multigrid.py:496-513).  The
oracle runs here only as the checker (test infrastructure).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402  (roofline model: SURVEY 8(d) fixed bytes / ops per DoF, measured peaks)
from oracle import oracle as O  # noqa: E402
from paper_2210_15280_b200 import CellILU, DevicePlan, _lib, fitting, lattice, stencil  # noqa: E402


def u0_for(level, seed):
    mask = lattice.interior_mask(level)
    u = np.zeros(lattice.grid_size(level))
    u[mask] = np.random.default_rng(seed).uniform(-1, 1, int(mask.sum()))
    return u


def gpu_run(plan, u0, f, sweeps):
    """(u after `sweeps`, rate, ms per sweep of the timed call)."""
    u = torch.as_tensor(u0, device="cuda")
    ft = torch.as_tensor(f, device="cuda")
    norms = [float(torch.linalg.norm(u))]
    for _ in range(sweeps - 1):
        plan.sweep(u, ft, 1)
        norms.append(float(torch.linalg.norm(u)))
    # timed: one more call of `sweeps` sweeps on a copy (includes the call's layout conversion)
    uc = u.clone()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    plan.sweep(uc, ft, sweeps)
    e1.record()
    torch.cuda.synchronize()
    plan.sweep(u, ft, 1)
    norms.append(float(torch.linalg.norm(u)))
    return u.cpu().numpy(), norms[-1] / norms[-2], e0.elapsed_time(e1) / sweeps


def oracle_run(fit, src, level, u0, f, sweeps):
    sur = O.OracleSurrogate(level, fit.lcoefs, fit.dcoefs, fit.variant, fit.band_ranks, fit.store_rows)
    u = u0.copy()
    norms = [float(np.linalg.norm(u))]
    for _ in range(sweeps):
        O.sweeps(sur, level, src.data, u, f, 1)
        norms.append(float(np.linalg.norm(u)))
    return u, norms[-1] / norms[-2]


def one(cfg, level, q, verts, coeff, sweeps, src=None, stored=False):
    t0 = time.time()
    src = src or stencil.stencil_source(verts, level, coeff)
    fit = fitting.fit_surrogate_ilu(src, level, (q, q, q), "v1")
    setup = time.time() - t0
    op = {"arow": src.data} if src.constant else {"arows": src.data}
    plan = DevicePlan(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows, **op)
    u0 = u0_for(level, cfg)
    f = np.zeros_like(u0)
    ug, rate, ms = gpu_run(plan, u0, f, sweeps)
    uo, rate_o = oracle_run(fit, src, level, u0, f, sweeps)
    N = lattice.interior_size(level)
    rec = {"config": cfg, "level": level, "q": q, "effective_degrees": list(fit.degrees), "sweeps": sweeps,
           "interior_dofs": N, "setup_s": round(setup, 1), "gpu_ms_per_sweep": ms,
           "gpu_dof_updates_per_s": N / (ms / 1e3), "rate_gpu": rate, "rate_oracle": rate_o,
           "rate_equal_3_digits": f"{rate:.3g}" == f"{rate_o:.3g}", "one_minus_rate": 1.0 - rate,
           "max_rel_err_vs_oracle": float(np.abs(ug - uo).max() / np.abs(uo).max()),
           "bitwise_vs_oracle": bool(np.array_equal(ug, uo)),
           "stencil": "constant row" if src.constant else "per-point rows"}
    bpd = bench.algo_bytes(level, "v1")["sweep"]
    opd = bench.algo_ops(level, fit.degrees)
    rt = bench.roofline_time(N, bpd, opd)
    t_roof = max(rt["t_hbm_s"], rt["t_fp64_s"])
    rec["roofline"] = {"bound": rt["bound"], "algorithmic_bytes_per_dof": bpd, "algorithmic_fp64_ops_per_dof": opd,
                       "t_roofline_ms": t_roof * 1e3, "frac": t_roof / (ms / 1e3), "hbm_gbs": rt["hbm_gbs"],
                       "fp64_tflops": rt["fp64_tflops"]}
    if stored:
        fr = fitting.factorize_tet(src, level, full_store=True)
        cplan = CellILU(fr).plan(**op)
        u = torch.as_tensor(u0, device="cuda")
        ft = torch.as_tensor(f, device="cuda")
        cplan.sweep(u, ft, 2, stored=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        cplan.sweep(u, ft, 5, stored=True)
        e1.record()
        torch.cuda.synchronize()
        sms = e0.elapsed_time(e1) / 5
        rec["stored_ilu_ms_per_sweep"] = sms
        rec["stored_ilu_dof_updates_per_s"] = N / (sms / 1e3)
        # K4: 48 B vectors + 7 L (fwd) + 7 transposed L and 1/D (bwd) = 168 B/DoF, 60 ops
        rk = bench.roofline_time(N, 168.0, 60.0)
        tk = max(rk["t_hbm_s"], rk["t_fp64_s"])
        rec["stored_ilu_roofline"] = {"bound": rk["bound"], "algorithmic_bytes_per_dof": 168.0,
                                      "t_roofline_ms": tk * 1e3, "frac": tk / (sms / 1e3)}
    return rec, src


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,5")
    ap.add_argument("--level5", type=int, default=8)
    args = ap.parse_args()
    want = {int(c) for c in args.configs.split(",")}
    out = {"device": torch.cuda.get_device_name(0), "records": []}
    if 1 in want:
        rec, _ = one(1, 5, 4, lattice.unit_tet(), stencil.CoefficientField.constant(1.0), 20, stored=True)
        out["records"].append(rec)
        print(json.dumps(rec), file=sys.stderr, flush=True)
    if 2 in want:
        rec, _ = one(2, 7, 6, lattice.distorted_tet(), stencil.diag_tensor((1.0, 1.0, 1e-3)), 50)
        out["records"].append(rec)
        print(json.dumps(rec), file=sys.stderr, flush=True)
    if 5 in want:
        L = args.level5
        t0 = time.time()
        src = stencil.stencil_source(lattice.distorted_tet(), L, stencil.diag_tensor((1.0, 1e-2, 1.0)))
        out["config5_stencil_setup_s"] = round(time.time() - t0, 1)
        for q in range(0, 9):
            rec, _ = one(5, L, q, None, None, 20, src=src, stored=(q in (0, 4, 8)))
            out["records"].append(rec)
            print(json.dumps(rec), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

"""Benchmark: surrogate ILU(0) smoother DoF-updates/s on B200 (BASELINE.json metric).

Default workload = configs[3]: the hybrid macro-mesh of 384 Kuhn macro-tets (4x4x4 unit
cubes x 6), each refined to level 7 (333,375 interior DoF per tet, 128,016,000 total),
Poisson, Dirichlet 0 on every macro-face, u ~ U[-1,1] (one global stream, seed 4, drawn in
(tet, interior rank) order), f = 0, surrogate degree q = 6 (effective (4,4,5)), variant V1.
It is the one configuration that spans 1-8 GPUs; the tets are partitioned contiguously
across ranks (one process per GPU) with a per-sweep residual-norm allreduce (NCCL).

One step = one smoothing sweep (residual, forward L solve, D^-1 + backward L^T solve,
update) over every tet of the rank, inputs resident in HBM (u, f are 1.1 GB each: larger
than L2, so no flush is needed).  `e2e` = the same metric through the public API with
pinned host buffers: H2D of u and f, `--e2e-sweeps` sweeps, D2H of u and the norms.

The line also carries `single_tet` (rank 0, N=1): one macro-tet at level 9 (configs[2] geometry
and size, k = 1) through the plane-layout band kernels -- the north star's single-tet target --
with its own roofline fraction, API-call time and e2e from pinned host buffers.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ILU(0) smoother DoF-updates/s (fwd+bwd sweep), 1–8 B200, % of roofline"
UNIT = "DoF-updates/s"
CFG4 = dict(tets=384, level=7, q=6, variant="v1", seed=4)
HBM_FALLBACK = 6650.0


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ----------------------------------------------------------------------------------------------
# distributed plumbing
# ----------------------------------------------------------------------------------------------
class Dist:
    def __init__(self, backend="nccl", init=True):
        import torch
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        self.torch = torch
        self.dist = None
        if self.world > 1 and init:
            import torch.distributed as dist
            if backend == "nccl":
                torch.cuda.set_device(self.local_rank)
            dist.init_process_group(backend)
            self.dist = dist

    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def max(self, x: float) -> float:
        if not self.dist:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t[0])

    def close(self):
        if self.dist:
            self.dist.destroy_process_group()


# ----------------------------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ----------------------------------------------------------------------------------------------
class Clocks:
    """SM clock and throttle reasons sampled DURING the timed region: NVML (pynvml) every 2 ms on a
    side thread (short timed regions still get samples); nvidia-smi -lms fallback."""
    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.sm: list[float] = []
        self.smax: list[float] = []
        self.mask = 0
        self.stop_ev = threading.Event()
        self.t = None
        self.nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            h = None
            try:
                import torch
                uuid = str(torch.cuda.get_device_properties(gpu).uuid)
                h = pynvml.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(gpu)
            self.nvml, self.h = pynvml, h
        except Exception:
            self.nvml = None

    def _sample(self):
        N, h = self.nvml, self.h
        self.sm.append(float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)))
        self.smax.append(float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)))
        try:
            self.mask |= int(N.nvmlDeviceGetCurrentClocksEventReasons(h))
        except AttributeError:
            self.mask |= int(N.nvmlDeviceGetCurrentClocksThrottleReasons(h))

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                self._sample()
            except Exception:
                return
            self.stop_ev.wait(0.002)

    def start(self):
        if self.nvml is None:
            return
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def stop(self) -> dict:
        if self.nvml is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"], "samples": 0}
        self.stop_ev.set()
        self.t.join(timeout=2)
        if not self.sm:
            self._sample()
        reasons = sorted(k for k, bit in self.REASONS.items() if self.mask & bit)
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": max(self.smax), "reasons": reasons,
                "samples": len(self.sm), "source": "NVML, 2 ms period, timed region"}


# ----------------------------------------------------------------------------------------------
# workload
# ----------------------------------------------------------------------------------------------
def draw_u0(level: int, first_tet: int, ntets: int, seed: int) -> np.ndarray:
    """u0 for tets [first_tet, first_tet + ntets) of one global U[-1,1] stream drawn in
    (tet, interior rank) order -- independent of the GPU count."""
    from paper_2210_15280_b200 import lattice
    mask = lattice.interior_mask(level)
    nint = int(mask.sum())
    rng = np.random.default_rng(seed)
    rng.bit_generator.advance(first_tet * nint)
    u = np.zeros((ntets, len(mask)))
    for t in range(ntets):
        u[t, mask] = rng.uniform(-1.0, 1.0, nint)
    return u


def peaks() -> dict:
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        return {}


def algo_bytes(level: int, nband: int, variant: str, shared_surrogate: bool = True) -> dict:
    """Algorithmic bytes per interior DoF.  "sweep" is SURVEY 8(d)'s fixed model (vectors once per
    pass, plus each tet's V1 band rows once per pass).  The per-kernel figures count what a kernel
    must move: the batched kernels share ONE band store among all tets of a group (read once per
    point, through the per-point coefficient table shared by every tet of the batch, L2-resident),
    so their per-DoF band share is ~0; the sentinel re-arm writes (8 B/DoF per pass) are an
    implementation overhead and are not counted."""
    from paper_2210_15280_b200 import lattice
    N = lattice.interior_size(level)
    band = 72.0 * nband / N if variant == "v1" else 0.0
    kb = 0.0 if shared_surrogate else band
    return {
        "sweep": 48.0 + 2 * band,
        "batch_fwd": 24.0 + kb, "batch_bwd": 24.0 + kb,      # fused passes: u,f -> w ; w,u -> u
        "residual": 24.0, "simple_fwd": 16.0 + band, "simple_bwd": 24.0 + band,
    }


def traffic_from_profiles(kernel: str):
    """dram bytes per launch of `kernel` from the committed ncu summary, or None."""
    try:
        tab = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        return tab.get(kernel)
    except (OSError, ValueError):
        return None


# ----------------------------------------------------------------------------------------------
# CPU baseline (oracle port) -- test infrastructure, never the product path
# ----------------------------------------------------------------------------------------------
def cpu_reference(fit, src, level: int, ntets_sample: int, threads: int, sweeps: int = 1) -> dict:
    from oracle import oracle as O
    from paper_2210_15280_b200 import lattice
    sur = O.OracleSurrogate(level, fit.lcoefs, fit.dcoefs, fit.variant, fit.band_ranks, fit.store_rows)
    u = draw_u0(level, 0, ntets_sample, CFG4["seed"])
    f = np.zeros_like(u)
    t0 = time.perf_counter()
    used = O.sweeps_many(sur, level, np.atleast_1d(src.data), u, f, sweeps, nthreads=threads)
    dt = time.perf_counter() - t0
    dofs = lattice.interior_size(level) * ntets_sample * sweeps
    return {"value": dofs / dt, "unit": UNIT, "cores": used, "kind": "port", "seconds": dt,
            "sample": f"{ntets_sample} Kuhn tets x {sweeps} sweep (L{level}, q=6 eff {tuple(fit.degrees)}, V1): "
                      f"oracle/tilu_oracle.c (serial C restatement of the reference Numba sweep), one OpenMP "
                      f"thread per tet"}


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def build_config4_fit():
    from paper_2210_15280_b200 import fitting, lattice, stencil
    src = stencil.stencil_source(lattice.kuhn_tet((0, 1, 2)), CFG4["level"], stencil.CoefficientField.constant(1.0))
    q = CFG4["q"]
    return src, fitting.fit_surrogate_ilu(src, CFG4["level"], (q, q, q), CFG4["variant"])


def run_reference(args, D: Dist):
    """--impl reference: the reference's CPU sweep (oracle port, all host threads), rank 0 only."""
    if D.rank != 0:
        return
    src, fit = build_config4_fit()
    threads = host_threads()
    nt = min(CFG4["tets"], max(threads, 8))
    for _ in range(args.warmup):
        cpu_reference(fit, src, CFG4["level"], nt, threads)
    vals = [cpu_reference(fit, src, CFG4["level"], nt, threads) for _ in range(args.steps)]
    secs = sum(v["seconds"] for v in vals)
    dofs_step = vals[0]["value"] * vals[0]["seconds"]
    value = dofs_step * len(vals) / secs
    cb = dict(vals[0])
    cb.pop("seconds")
    cb["value"] = value
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / len(vals),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(fit, 1, extra={"sample_tets_per_step": nt}),
        "cpu_baseline": cb, "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_block(fit, world, extra=None) -> dict:
    from paper_2210_15280_b200 import lattice
    c = {
        "workload": "configs[3]: 384 Kuhn macro-tets (4x4x4 unit cubes x 6), level 7 each, Poisson, "
                    "Dirichlet 0, u~U[-1,1] seed 4, f=0, q=6, V1; one step = one sweep over all tets",
        "tets": CFG4["tets"], "level": CFG4["level"], "dofs": CFG4["tets"] * lattice.interior_size(CFG4["level"]),
        "q": CFG4["q"], "effective_degrees": list(fit.degrees), "variant": CFG4["variant"],
        "parallelism": f"macro-tet partition x{world}, NCCL residual-norm allreduce per sweep",
        "l2": "inputs larger than L2 (u, f 1.1 GB each); no flush needed",
    }
    if extra:
        c.update(extra)
    return c


# ----------------------------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------------------------
def run_single(args) -> dict:
    """One macro-tet at the north star's level (configs[2] geometry and size: unit tet, level 9,
    q = 6 -> effective (4, 4, 4), V1, f ~ N(0, 1), u = 0) through the plane-layout band kernels.
    The coefficient is k = 1 (constant stencil): config 3's variable k(x) needs the per-point
    stencil assembled on the host (28 min in the reference) and a per-point residual; the sweep
    kernels are the same.  Reported: device time per sweep of the two plane kernels (resident,
    `value`), the API call time (pack + sweeps + unpack + norms per call), and e2e from pinned host
    buffers (H2D u, f -> sweeps -> D2H u)."""
    import torch

    from paper_2210_15280_b200 import DevicePlan, _lib, fitting, lattice, stencil
    level, q, sweeps = args.single_level, 6, args.single_sweeps
    t0 = time.time()
    src = stencil.stencil_source(lattice.unit_tet(), level, stencil.CoefficientField.constant(1.0))
    fit = fitting.fit_surrogate_ilu(src, level, (q, q, q), "v1")
    setup_s = time.time() - t0
    N = lattice.interior_size(level)
    mask = lattice.interior_mask(level)
    f_host = np.zeros(lattice.grid_size(level))
    f_host[mask] = np.random.default_rng(3).normal(size=int(mask.sum()))
    dev = torch.device("cuda", torch.cuda.current_device())
    p = DevicePlan(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows, arow=src.data,
                   fast=args.fast)
    f = torch.as_tensor(f_host, device=dev)
    u = torch.zeros_like(f)
    p.sweep(u, f, 3)  # warm-up (workspace, arming, clocks)
    torch.cuda.synchronize()
    u.zero_()
    _lib.profile_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rn = p.sweep(u, f, sweeps, norms=True)
    e1.record()
    torch.cuda.synchronize()
    kprof = _lib.profile_read()
    _lib.profile_enable(False)
    call_ms = e0.elapsed_time(e1) / sweeps
    kern_ms = sum(tot for name, (cnt, tot) in kprof.items() if name in ("plane_fwd", "plane_bwd")) / sweeps
    ab = algo_bytes(level, len(fit.band_ranks), "v1")["sweep"]
    pk = peaks()
    peak = pk.get("hbm_gbs") or HBM_FALLBACK
    achieved = ab * N / (kern_ms / 1e3) / 1e9
    # e2e: pinned host u, f -> device -> sweeps -> host u
    uh = torch.zeros(f.numel(), dtype=torch.float64).pin_memory()
    fh = torch.from_numpy(f_host).pin_memory()
    torch.cuda.synchronize()
    e0.record()
    ud = uh.to(dev, non_blocking=True)
    fd = fh.to(dev, non_blocking=True)
    p.sweep(ud, fd, sweeps)
    uh.copy_(ud, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    rho = float((rn[-1] / rn[-2]).sqrt()) if sweeps >= 2 else None
    return {
        "workload": f"configs[2] geometry/size with k=1: unit macro-tet, level {level} ({N} interior DoF), "
                    f"q=6 eff {tuple(fit.degrees)}, V1, f~N(0,1) seed 3, u=0, {sweeps} sweeps per call",
        "value": N / (kern_ms / 1e3), "unit": UNIT, "ms_per_sweep_kernels": kern_ms,
        "ms_per_sweep_call": call_ms, "api_value": N / (call_ms / 1e3),
        "roofline": {"bound": "hbm", "algorithmic_bytes_per_dof": ab, "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak},
        "e2e": {"value": N * sweeps / (e2e_ms / 1e3), "unit": UNIT, "ms": e2e_ms,
                "h2d_bytes_per_step": 2 * f.numel() * 8, "d2h_bytes_per_step": f.numel() * 8,
                "sweeps_per_step": sweeps, "api": "DevicePlan.sweep on device copies of pinned host u, f"},
        "kernels": {k: {"launches": c, "avg_ms": t / c} for k, (c, t) in kprof.items()},
        "residual_ratio_last": rho, "setup_s": setup_s,
        "mode": "fast (FMA)" if args.fast else "exact (bitwise)",
    }


def run_ours(args, D: Dist):
    import torch

    from paper_2210_15280_b200 import MacroMeshSmoother, _lib, lattice, stencil
    from paper_2210_15280_b200.partition import partition

    dev = torch.device("cuda", D.local_rank)
    torch.cuda.set_device(dev)
    level = CFG4["level"]
    t0 = time.time()
    tets = lattice.kuhn_mesh(4)
    q = CFG4["q"]
    mm = MacroMeshSmoother(tets, level, stencil.CoefficientField.constant(1.0), (q, q, q), CFG4["variant"],
                           rank=D.rank, world_size=D.world, fast=args.fast, simple=args.simple)
    fit = mm.smoothers[0].precond
    local = partition(CFG4["tets"], D.world)[D.rank]
    u_host = draw_u0(level, local.start, len(local), CFG4["seed"])
    u0 = torch.as_tensor(u_host, device=dev)
    u = u0.clone()
    f = torch.zeros_like(u)
    log(f"[rank {D.rank}] setup {time.time() - t0:.1f}s: {len(local)} tets, groups={len(mm.groups)}, "
        f"eff degrees {fit.degrees}")

    # resident packed state (inputs in HBM before the timed region)
    mm.load(u, f)
    for _ in range(args.warmup):
        mm.sweep(1)
    torch.cuda.synchronize()

    # timed region: K sweeps, kernel events on
    _lib.profile_enable(True)
    mm.launches = 0
    clocks = Clocks(D.local_rank)
    D.barrier()
    torch.cuda.synchronize()
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    norms = []
    for _ in range(args.steps):
        norms.append(mm.sweep(1))
    ev1.record()
    torch.cuda.synchronize()
    D.barrier()
    clk = clocks.stop()
    ms_local = ev0.elapsed_time(ev1)
    kprof = _lib.profile_read()
    _lib.profile_enable(False)
    launches = mm.launches
    ms = D.max(ms_local)
    dofs_total = CFG4["tets"] * lattice.interior_size(level)
    value = dofs_total * args.steps / (ms / 1e3)

    # dominant kernel roofline
    ab = algo_bytes(level, len(fit.band_ranks), CFG4["variant"])
    pk = peaks()
    peak = pk.get("hbm_gbs") or HBM_FALLBACK
    dom = max(kprof.items(), key=lambda kv: kv[1][1]) if kprof else None
    roof = None
    if dom is not None:
        name, (cnt, tot) = dom
        per_launch_ms = tot / cnt
        bytes_per_launch = ab.get(name, ab["sweep"]) * lattice.interior_size(level) * len(local)
        achieved = bytes_per_launch / (per_launch_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": name, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic_from_profiles(name),
                "algorithmic_bytes_per_launch": bytes_per_launch, "avg_launch_ms": per_launch_ms,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (of measured)" if pk.get("hbm_gbs") else
                               "B200_PROFILING.md fallback (of fallback)",
                "step_share": tot / ms_local if ms_local else None}
    sweep_ms = ms / args.steps
    sweep_achieved = ab["sweep"] * dofs_total / D.world / (sweep_ms / 1e3) / 1e9
    kernels = {k: {"launches": c, "avg_ms": t / c} for k, (c, t) in kprof.items()}

    # e2e through the public API with pinned host buffers
    e2e = None
    if args.e2e_sweeps > 0:
        uh = torch.from_numpy(u_host).pin_memory()
        fh = torch.zeros_like(uh).pin_memory()
        mm.apply_host(uh.clone().pin_memory(), fh, args.e2e_sweeps, chunk=args.e2e_chunk)  # warm
        torch.cuda.synchronize()
        D.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(1, min(args.steps, 3))
        e0.record()
        for _ in range(reps):
            mm.apply_host(uh, fh, args.e2e_sweeps, chunk=args.e2e_chunk)
        e1.record()
        torch.cuda.synchronize()
        D.barrier()
        ems = D.max(e0.elapsed_time(e1)) / reps
        h2d = 2 * uh.numel() * 8
        d2h = uh.numel() * 8 + 8 * args.e2e_sweeps
        e2e = {"value": dofs_total * args.e2e_sweeps / (ems / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": h2d * D.world, "d2h_bytes_per_step": d2h * D.world,
               "sweeps_per_step": args.e2e_sweeps, "ms_per_step": ems,
               "api": f"MacroMeshSmoother.apply_host(pinned u, f, sweeps): {args.e2e_chunk}-tet chunks "
                      f"pipelined on 2 streams (H2D / sweeps / D2H overlap)"}

    # CPU baseline (rank 0, N=1 only)
    cpu = None
    if D.world == 1 and D.rank == 0 and not args.no_cpu:
        threads = host_threads()
        src = mm.smoothers[0].source
        nt = min(CFG4["tets"], max(threads, 8))
        cpu = cpu_reference(fit, src, level, nt, threads)
        cpu.pop("seconds")

    single = None
    if D.world == 1 and D.rank == 0 and not args.no_single:
        try:
            single = run_single(args)
        except Exception as e:  # reported, never silently replaced by another path
            single = {"error": f"{type(e).__name__}: {e}"}

    if D.rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": D.world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_block(fit, D.world, {"mode": "fast (FMA)" if args.fast else "exact (bitwise)",
                                                  "schedule": "simple" if args.simple else "auto"}),
            "roofline": roof,
            "sweep_roofline": {"bound": "hbm", "algorithmic_bytes_per_dof": ab["sweep"], "achieved": sweep_achieved,
                               "peak": peak, "unit": "GB/s", "frac": sweep_achieved / peak},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "kernels": kernels, "clocks": clk,
            "residual_norm2_last": float(norms[-1][-1]) if norms else None,
            "single_tet": single,
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--e2e-sweeps", type=int, default=3)
    ap.add_argument("--e2e-chunk", type=int, default=64, help="tets per pipelined host<->device chunk")
    ap.add_argument("--fast", action="store_true", help="FMA substitution (<=1e-12, not bitwise)")
    ap.add_argument("--simple", action="store_true", help="force the reference-layout kernels")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--no-single", action="store_true", help="skip the single-macro-tet (level 9) leg")
    ap.add_argument("--single-level", type=int, default=9)
    ap.add_argument("--single-sweeps", type=int, default=100)
    args = ap.parse_args()
    if args.warmup < 3:
        log("note: warmup raised to 3 (timing rules)")
        args.warmup = 3
    # the reference arm runs on rank 0 only and needs no process group
    D = Dist("nccl", init=args.impl == "ours")
    try:
        if args.impl == "reference":
            run_reference(args, D)
        else:
            run_ours(args, D)
    finally:
        D.close()


if __name__ == "__main__":
    main()

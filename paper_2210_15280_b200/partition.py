"""Macro-tet partitioning across GPUs (config 4: 384 Kuhn macro-tets on 1-8 B200).

Macro-tets with Dirichlet data on every macro-face are independent units: the
reference's cell stage is block-Jacobi across cells (multigrid.py:419-429), so the
sweep itself needs no halo exchange.  Each rank (one process per GPU) owns a
contiguous block of tets; the only collective is the per-sweep residual-norm
allreduce (one fp64 per sweep, NCCL over NVLink/NVSwitch), enqueued on a side
stream so it overlaps the next sweep.
"""

from __future__ import annotations

import hashlib

import numpy as np

from . import lattice
from .smoother import SmootherConfig, SurrogateILUSmoother
from .stencil import CoefficientField, stencil_source

try:
    import torch
    import torch.distributed as dist
except ImportError:  # pragma: no cover
    torch = dist = None


def partition(ntets: int, world_size: int) -> list[range]:
    """Contiguous blocks, sizes differing by at most one (equal DoF per tet -> balanced)."""
    if world_size < 1 or ntets < 0:
        raise ValueError("world_size >= 1 and ntets >= 0 required")
    base, extra = divmod(ntets, world_size)
    out, start = [], 0
    for r in range(world_size):
        size = base + (1 if r < extra else 0)
        out.append(range(start, start + size))
        start += size
    return out


def group_by_operator(rows: list[np.ndarray]) -> list[list[int]]:
    """Indices of tets whose operator rows are bitwise identical share one surrogate."""
    groups: dict[bytes, list[int]] = {}
    for i, r in enumerate(rows):
        groups.setdefault(hashlib.sha1(np.ascontiguousarray(r).tobytes()).digest(), []).append(i)
    return list(groups.values())


def allreduce_norms(local: "torch.Tensor", group=None) -> "torch.Tensor":
    """Sum of per-rank residual norm^2 (in place); a no-op on one rank."""
    if dist is not None and dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(local, op=dist.ReduceOp.SUM, group=group)
    return local


class SweepNorms:
    """Per-sweep global residual norm^2 of a macro-mesh: each rank adds its tets' ||r||^2 (fixed
    order: groups in order, tets in order within a group's per-tet vector), then one allreduce per
    sweep.  On CUDA tensors the allreduce of sweep k is enqueued on a side stream that waits only
    for sweep k, so it overlaps sweep k+1; on CPU tensors (gloo) it runs inline."""

    def __init__(self, sweeps: int, device, group=None):
        self.norms = torch.zeros(sweeps, dtype=torch.float64, device=device)
        self.group = group
        self.side = None
        if self.norms.is_cuda:
            self.side = torch.cuda.Stream(device=self.norms.device)

    def add(self, k: int, per_tet: "torch.Tensor") -> None:
        self.norms[k] += per_tet.sum()

    def close_sweep(self, k: int) -> None:
        if self.side is None:
            allreduce_norms(self.norms[k:k + 1], self.group)
            return
        ev = torch.cuda.Event()
        ev.record()
        with torch.cuda.stream(self.side):
            self.side.wait_event(ev)
            allreduce_norms(self.norms[k:k + 1], self.group)

    def result(self, check_finite: bool = False) -> "torch.Tensor":
        """The allreduced per-sweep norms; ``check_finite`` (synchronises) raises FloatingPointError on NaN / inf."""
        if self.side is not None:
            torch.cuda.current_stream(self.norms.device).wait_stream(self.side)
        if check_finite and not bool(torch.isfinite(self.norms).all()):
            k = int(torch.nonzero(~torch.isfinite(self.norms))[0])
            raise FloatingPointError(f"non-finite global residual norm before sweep {k}")
        return self.norms


class MacroMeshSmoother:
    """Smoother over this rank's share of a macro-mesh of independent macro-tets."""

    def __init__(self, tets: list[np.ndarray], level: int, coeff: CoefficientField | None = None,
                 degrees=(6, 6, 6), variant: str = "v1", rank: int = 0, world_size: int = 1, group=None,
                 fast: bool = False, simple: bool = False):
        self.level = level
        self.grid = lattice.grid_size(level)
        self.ntets_global = len(tets)
        self.local = partition(len(tets), world_size)[rank]
        self.group = group
        coeff = coeff or CoefficientField.constant(1.0)
        sources = [stencil_source(tets[i], level, coeff) for i in self.local]
        self.groups = group_by_operator([s.data for s in sources])
        self.smoothers = [SurrogateILUSmoother(sources[g[0]], level, SmootherConfig(
            "surrogate_ilu", tuple(degrees), variant), fast=fast, simple=simple) for g in self.groups]
        self._agg = None
        self.launches = 0   # kernels enqueued by apply() so far (bench accounting)

    @property
    def ntets_local(self) -> int:
        return len(self.local)

    def apply(self, u: "torch.Tensor", f: "torch.Tensor", sweeps: int = 1, residual_norms: bool = True):
        """u, f: this rank's tets [ntets_local, grid] (CUDA fp64).  Returns the global
        ||f - A u||^2 before each sweep ([sweeps], summed over all ranks) if requested."""
        if u.shape != (self.ntets_local, self.grid):
            raise ValueError(f"u must be [{self.ntets_local}, {self.grid}]")
        agg = SweepNorms(sweeps, u.device, self.group) if residual_norms else None
        views = []
        for g, sm in zip(self.groups, self.smoothers):
            contiguous = g == list(range(g[0], g[0] + len(g)))
            views.append((sm, g, contiguous))
        for k in range(sweeps):
            for sm, g, contiguous in views:
                if contiguous:
                    rn = sm.apply(u[g[0]:g[0] + len(g)], f[g[0]:g[0] + len(g)], 1,
                                  residual_norms=residual_norms)
                else:
                    idx = torch.as_tensor(g, device=u.device)
                    ug = u.index_select(0, idx).contiguous()
                    rn = sm.apply(ug, f.index_select(0, idx).contiguous(), 1, residual_norms=residual_norms)
                    u.index_copy_(0, idx, ug)
                self.launches += sm.plan.last_launch_count()
                if agg is not None:
                    agg.add(k, rn)
            if agg is not None:
                agg.close_sweep(k)   # overlaps the next sweep (side stream)
        return agg.result() if agg is not None else None

    # -- resident packed state (the hot path of the benchmark) ----------------------------------
    def load(self, u: "torch.Tensor", f: "torch.Tensor") -> None:
        """Move this rank's tets [ntets_local, grid] into the packed, interleaved device layout."""
        self._res = []
        for g, sm in zip(self.groups, self.smoothers):
            idx = torch.as_tensor(g, device=u.device)
            ug, fg = u.index_select(0, idx).contiguous(), f.index_select(0, idx).contiguous()
            p = sm.plan
            up, fp = p.pack(ug), p.pack(fg)
            wp = p.new_scratch(len(g), device=up.device)
            self._res.append((sm, g, up, fp, wp))

    def sweep(self, sweeps: int = 1, residual_norms: bool = True):
        """``sweeps`` fused sweeps on the resident packed state; per-sweep global ||r||^2 is
        allreduced on a side stream (overlapping the next sweep)."""
        dev = self._res[0][2].device
        if residual_norms and (self._agg is None or len(self._agg.norms) != sweeps):
            self._agg = SweepNorms(sweeps, dev, self.group)
        agg = self._agg if residual_norms else None
        if agg is not None:
            agg.norms = torch.zeros(sweeps, dtype=torch.float64, device=dev)
        for k in range(sweeps):
            for sm, g, up, fp, wp in self._res:
                rn = sm.plan.sweep_packed(up, fp, wp, len(g), 1, norms=residual_norms)
                self.launches += sm.plan.last_launch_count()
                if agg is not None:
                    agg.add(k, rn)
            if agg is not None:
                agg.close_sweep(k)
        return agg.result() if agg is not None else None

    def store(self, u: "torch.Tensor") -> "torch.Tensor":
        """Unpack the resident state back into u [ntets_local, grid] (reference layout)."""
        for sm, g, up, fp, wp in self._res:
            idx = torch.as_tensor(g, device=u.device)
            ug = torch.empty((len(g), self.grid), dtype=u.dtype, device=u.device)
            sm.plan.unpack(up, ug)
            u.index_copy_(0, idx, ug)
        return u

    def apply_host(self, u_host: "torch.Tensor", f_host: "torch.Tensor", sweeps: int = 1,
                   residual_norms: bool = True, chunk: int = 64):
        """End-to-end call on (pinned) host tensors [ntets_local, grid]: H2D of u and f, ``sweeps``
        sweeps, D2H of u (in place) and of the global norms.  Returns the norms (host tensor) or None.

        Pipelined: the tets go through in chunks of ``chunk`` (independent packed groups) on two
        streams, so the H2D of one chunk and the D2H of another overlap the sweeps of a third."""
        dev = torch.device("cuda", torch.cuda.current_device())
        main = torch.cuda.current_stream(dev)
        if getattr(self, "_copy_streams", None) is None:
            self._copy_streams = [torch.cuda.Stream(device=dev) for _ in range(2)]
            self._scratch = {}
        parts = []  # (smoother index, first tet, count): host-contiguous runs cut into chunks
        for si, g in enumerate(self.groups):
            run0 = 0
            for i in range(1, len(g) + 1):
                if i == len(g) or g[i] != g[i - 1] + 1:
                    for a in range(g[run0], g[i - 1] + 1, chunk):
                        parts.append((si, a, min(chunk, g[i - 1] + 1 - a)))
                    run0 = i
        pn = torch.zeros((len(parts), sweeps), dtype=torch.float64, device=dev) if residual_norms else None
        start = torch.cuda.Event()
        start.record(main)
        for i, (si, a, cnt) in enumerate(parts):
            s = self._copy_streams[i % 2]
            s.wait_event(start)
            p = self.smoothers[si].plan
            with torch.cuda.stream(s):
                uc = u_host[a:a + cnt].to(dev, non_blocking=True)
                fc = f_host[a:a + cnt].to(dev, non_blocking=True)
                up, fp = p.pack(uc), p.pack(fc)
                key = (si, cnt, i % 2)
                if key not in self._scratch:
                    self._scratch[key] = p.new_scratch(cnt, device=dev)
                rn = p.sweep_packed(up, fp, self._scratch[key], cnt, sweeps, norms=residual_norms)
                self.launches += p.last_launch_count() + 3  # + pack u, pack f, unpack
                p.unpack(up, uc)
                u_host[a:a + cnt].copy_(uc, non_blocking=True)
                if residual_norms:
                    pn[i] = rn.sum(dim=1)
        for s in self._copy_streams:
            main.wait_stream(s)
        out = None
        if residual_norms:
            norms = pn.sum(dim=0)
            allreduce_norms(norms, self.group)
            out = norms.to("cpu", non_blocking=True)
        main.synchronize()
        return out

"""CPU-side checks: lattice conventions, the C-ABI library loads and exports every
symbol include/tilu.h declares, argument validation fails loudly, partitioner and the
residual-norm allreduce over gloo with world_size 2."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT, gpu_available
from paper_2210_15280_b200 import _lib, lattice
from paper_2210_15280_b200.partition import allreduce_norms, group_by_operator, partition


@pytest.mark.parametrize("level,grid,inner,nband", [(5, 6545, 4495, 1570), (7, 366145, 333375, 30754),
                                                    (8, 2862209, 2731135, 127010)])
def test_lattice_sizes(level, grid, inner, nband):
    """SURVEY.md 8(a) size table."""
    assert lattice.grid_size(level) == grid
    assert lattice.interior_size(level) == inner
    assert int(lattice.interior_mask(level).sum()) == inner
    assert len(lattice.band_ranks(level)) == nband


def test_rank_tables_roundtrip():
    L = 4
    coords = lattice.lattice_coords(L)
    assert np.array_equal(lattice.lattice_rank(coords, L), np.arange(len(coords)))
    ro = lattice.rank_tables(L)
    assert all(ro[z, y] + x == r for r, (x, y, z) in enumerate(coords))


def test_kuhn_mesh_config4():
    tets = lattice.kuhn_mesh(4)
    assert len(tets) == 384
    vol = [abs(np.linalg.det(t[1:] - t[0])) / 6 for t in tets]
    np.testing.assert_allclose(vol, 1 / 6)


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "tilu.h")).read()
    return sorted(set(re.findall(r"\b(tilu_[a-z0-9_]+)\s*\(", src)))


def test_abi_exports_every_declared_symbol():
    L = _lib.lib()
    declared = _declared_symbols()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(L, name), name
    assert set(_lib.EXPORTS) == set(declared)
    assert L.tilu_version() >= 100


def test_abi_rejects_bad_descriptors_without_crashing():
    import ctypes
    L = _lib.lib()
    h = ctypes.c_void_p()
    d = _lib.TiluDesc()
    d.level = 1
    assert L.tilu_plan_create(ctypes.byref(d), ctypes.byref(h)) == _lib.TILU_EINVAL
    assert b"level" in L.tilu_last_error()
    d.level, d.kx1, d.ky1, d.kz1, d.variant = 4, 10, 1, 1, 1
    assert L.tilu_plan_create(ctypes.byref(d), ctypes.byref(h)) == _lib.TILU_EUNSUPPORTED
    # null plan on every compute entry point: status code, no crash
    assert L.tilu_solve_into(None, None, 1, None) == _lib.TILU_EINVAL
    assert L.tilu_sweep(None, None, None, 1, 1, None, None) == _lib.TILU_EINVAL


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU failure path")
def test_no_cpu_fallback():
    """Without a GPU the product raises instead of computing on the CPU."""
    from paper_2210_15280_b200 import SurrogateILUSmoother
    with pytest.raises(Exception):
        SurrogateILUSmoother.setup(lattice.unit_tet(), 3, (1, 1, 1))


def test_partition_blocks():
    for n, w in [(384, 1), (384, 2), (384, 8), (10, 3), (3, 4)]:
        parts = partition(n, w)
        assert len(parts) == w
        assert [i for p in parts for i in p] == list(range(n))
        sizes = [len(p) for p in parts]
        assert max(sizes) - min(sizes) <= 1


def test_group_by_operator():
    a, b = np.arange(15.0), np.arange(15.0) + 1
    assert group_by_operator([a, b, a.copy(), b]) == [[0, 2], [1, 3]]


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    parts = partition(384, world)
    # each rank's local residual norm^2 = sum over its tets of (tet index + 1)
    local = torch.tensor([float(sum(i + 1 for i in parts[rank]))], dtype=torch.float64)
    allreduce_norms(local)
    q.put((rank, float(local[0]), list(parts[rank])[:1]))
    dist.destroy_process_group()


def test_allreduce_norms_gloo_world2():
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    total = 384 * 385 / 2
    assert out[0][1] == total and out[1][1] == total
    assert out[0][2] == [0] and out[1][2] == [192]


def _sweepnorms_worker(rank, world, port, q):
    """One rank of config 4's macro-mesh (level 3 here): per-tet residual norms of its own tets
    (C oracle sweeps), aggregated by MacroMeshSmoother's SweepNorms (fixed-order local sum + one
    allreduce per sweep) over gloo."""
    import torch
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2210_15280_b200 import fitting, lattice, stencil
    from paper_2210_15280_b200.partition import SweepNorms
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    level, sweeps = 3, 3
    src = stencil.stencil_source(lattice.kuhn_tet((0, 1, 2)), level, stencil.CoefficientField.constant(1.0))
    fit = fitting.fit_surrogate_ilu(src, level, (2, 2, 2), "v1")
    sur = O.OracleSurrogate(level, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows)
    mask = lattice.interior_mask(level)
    agg = SweepNorms(sweeps, "cpu")
    local = partition(384, world)[rank]
    per_tet = np.zeros((sweeps, len(local)))
    for i, t in enumerate(local):
        u = np.zeros(lattice.grid_size(level))
        u[mask] = np.random.default_rng(1000 + t).uniform(-1, 1, int(mask.sum()))
        per_tet[:, i] = O.sweeps(sur, level, src.data, u, np.zeros_like(u), sweeps, return_norms=True)
    for k in range(sweeps):
        agg.add(k, torch.as_tensor(per_tet[k]))
        agg.close_sweep(k)
    q.put((rank, agg.result().tolist(), per_tet.sum(axis=1).tolist()))
    dist.destroy_process_group()


def test_macro_mesh_norm_aggregation_gloo_world2():
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_sweepnorms_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g0, g1 = np.array(out[0][1]), np.array(out[1][1])
    want = np.array(out[0][2]) + np.array(out[1][2])
    assert np.array_equal(g0, g1)                     # every rank holds the same global norms
    np.testing.assert_allclose(g0, want, rtol=1e-14)  # = sum over all 384 tets' norms
    assert np.all(np.diff(g0) < 0)                     # the smoother decreases the residual


def test_sweep_norms_check_finite_cpu():
    import torch

    from paper_2210_15280_b200.partition import SweepNorms
    agg = SweepNorms(2, torch.device("cpu"))
    agg.add(0, torch.tensor([1.0, 2.0], dtype=torch.float64))
    agg.add(1, torch.tensor([float("nan"), 2.0], dtype=torch.float64))
    assert float(agg.result()[0]) == 3.0
    with pytest.raises(FloatingPointError):
        agg.result(check_finite=True)

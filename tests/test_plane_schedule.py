"""CPU checks of the single-tet plane kernels' band-task schedule (tilu_plane.cu make_tasks via the
C ABI): every interior row belongs to exactly one task, and the task order is topological for the
forward pass (a band task waits for the band below and the chunk below) and, reversed, for the
backward pass -- the property that makes the persistent-CTA ticket schedule deadlock-free."""

import pytest

from paper_2210_15280_b200 import _lib, lattice

PW = 4  # diagonals per band (tilu_plane.cu)


@pytest.mark.parametrize("level", [3, 4, 5, 6, 7, 8, 9])
def test_tasks_cover_rows_once(level):
    n = 2 ** level
    tasks = _lib.plane_tasks(level)
    assert len(tasks) == len(set(tasks))
    covered = {}
    for b, c in tasks:
        s0, z0 = 2 + PW * b, 1 + 32 * c
        for s in range(s0, s0 + PW):
            if s > n - 2:
                continue
            for z in range(z0, z0 + 32):
                if 1 <= z <= s - 1:
                    covered[(z, s - z)] = covered.get((z, s - z), 0) + 1
    rows = {(z, y) for z in range(1, n - 2) for y in range(1, n - 1 - z)}
    assert set(covered) == rows
    assert all(v == 1 for v in covered.values())
    assert sum(n - 1 - z - y for z, y in rows) == lattice.interior_size(level)


@pytest.mark.parametrize("level", [4, 6, 8, 9])
def test_order_is_topological_both_passes(level):
    tasks = _lib.plane_tasks(level)
    pos = {t: i for i, t in enumerate(tasks)}
    for (b, c), i in pos.items():
        # forward: band b-1 (same chunk and the chunk below), chunk c-1 of the same band
        for dep in ((b - 1, c), (b - 1, c - 1), (b, c - 1)):
            if dep in pos:
                assert pos[dep] < i, ((b, c), dep)
        # backward (reversed order): band b+1 (same chunk and the chunk above), chunk c+1
        for dep in ((b + 1, c), (b + 1, c + 1), (b, c + 1)):
            if dep in pos:
                assert pos[dep] > i, ((b, c), dep)

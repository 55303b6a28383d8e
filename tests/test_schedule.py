"""CPU verification of the batched path's wavefront schedule exactly as libtilu computes it:
every lower-neighbour dependency is produced early enough (same row: 1 step; same layer: a
full synchronisation window; layer below: D + 1 steps), a warp owns one row at a time, and
the window-by-window progress handoff completes (no deadlock) forward and backward."""

import numpy as np
import pytest

from paper_2210_15280_b200 import _lib

LOWER = [(-1, 0, 0), (0, -1, 0), (1, -1, 0), (-1, 1, -1), (0, 1, -1), (0, 0, -1), (1, 0, -1)]
BW = 8


def steps(level):
    s = _lib.batch_schedule(level)
    n = 2 ** level
    T = {}
    for zi in range(n - 3):
        z = zi + 1
        for y in range(1, n - 1 - z):
            for x in range(1, n - z - y):
                T[(x, y, z)] = int(s["O"][zi] + s["A"][zi] * (y - 1) + x - 1)
    return s, T


@pytest.mark.parametrize("level", [2, 3, 4, 5, 6])
def test_dependencies_respected(level):
    s, T = steps(level)
    D = s["D"]
    for (x, y, z), t in T.items():
        for dx, dy, dz in LOWER:
            q = (x + dx, y + dy, z + dz)
            if q not in T:
                continue
            lag = t - T[q]
            if dz == 0 and dy == 0:
                assert lag >= 1
            elif dz == 0:
                assert lag >= s["B"][z - 1], ((x, y, z), q)
            else:
                assert lag >= D + 1, ((x, y, z), q)
    assert max(T.values()) == s["Tmax"]


@pytest.mark.parametrize("level", [3, 5, 7, 9])
def test_one_row_per_warp(level):
    s = _lib.batch_schedule(level)
    n = 2 ** level
    for zi in range(n - 3):
        R = n - 2 - (zi + 1)
        assert s["A"][zi] >= 2 and s["A"][zi] * BW >= R and s["B"][zi] == s["A"][zi] - 1


def _simulate(s, n, backward):
    nl = n - 3
    Tmax, D = s["Tmax"], s["D"]
    lo = [int(Tmax - s["T1"][z]) if backward else int(s["O"][z]) for z in range(nl)]
    hi = [int(Tmax - s["O"][z]) if backward else int(s["T1"][z]) for z in range(nl)]
    prog, pos, done = [-1] * nl, list(lo), set()
    order = range(nl - 1, -1, -1) if backward else range(nl)
    moved = True
    while moved:
        moved = False
        for z in order:
            if z in done:
                continue
            dep = z + 1 if backward else z - 1
            B = int(s["B"][z])
            if 0 <= dep < nl and prog[dep] < min(pos[z] + B - 2 - D, hi[dep]):
                continue
            t1 = min(pos[z] + B, hi[z] + 1)
            prog[z], pos[z], moved = t1 - 1, t1, True
            if t1 > hi[z]:
                done.add(z)
    return len(done) == nl


@pytest.mark.parametrize("level", [2, 3, 4, 5, 6, 7, 8, 9])
def test_handoff_completes(level):
    s = _lib.batch_schedule(level)
    n = 2 ** level
    assert _simulate(s, n, backward=False)
    assert _simulate(s, n, backward=True)

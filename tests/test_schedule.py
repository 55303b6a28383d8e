"""CPU verification of the batched path's greedy wavefront schedule exactly as libtilu
computes it (tilu_batch_schedule): every value a point reads -- including the one-point-ahead
prefetch -- was produced in a synchronisation window already closed (same layer) or covered by
the progress counter the window waits for (layer below); rows of one warp never overlap; the
window-by-window progress handoff completes forward and backward (no deadlock)."""

import numpy as np
import pytest

from paper_2210_15280_b200 import _lib

LOWER = [(-1, 0, 0), (0, -1, 0), (1, -1, 0), (-1, 1, -1), (0, 1, -1), (0, 0, -1), (1, 0, -1)]


def row_id(n, z, y):
    return (z - 1) * (n - 2) - (z - 1) * z // 2 + (y - 1)


def schedule(level, bwin, pf=1):
    s = _lib.batch_schedule(level, bwin, pf)
    n = 2 ** level
    T = {}
    for z in range(1, n - 2):
        for y in range(1, n - 1 - z):
            st = int(s["start"][row_id(n, z, y)])
            for x in range(1, n - z - y):
                T[(x, y, z)] = st + x - 1
    T0 = {z: min(int(s["start"][row_id(n, z, y)]) for y in range(1, n - 1 - z)) for z in range(1, n - 2)}
    return s, T, T0


def window_start(t, t0, bwin):
    return t0 + ((t - t0) // bwin) * bwin


WP = [(4, 3), (1, 1), (2, 1), (8, 1), (4, 0)]


@pytest.mark.parametrize("bwin,pf", WP)
@pytest.mark.parametrize("level", [2, 3, 4, 5, 6])
def test_forward_reads_are_safe(level, bwin, pf):
    s, T, T0 = schedule(level, bwin, pf)
    n = 2 ** level
    D = s["D"]
    for (x, y, z), t in T.items():
        # points 1..pf are loaded at the row's first step, later ones pf steps ahead
        load_t = t - x + 1 if x <= pf else t - pf
        ws = window_start(load_t, T0[z], bwin)
        for dx, dy, dz in LOWER:
            q = (x + dx, y + dy, z + dz)
            if q not in T:
                continue
            tq = T[q]
            if dz == 0 and dy == 0:
                assert tq == t - 1                      # own row: register
            elif dz == 0:
                assert tq < ws, ((x, y, z), q)          # closed window of this CTA
            else:
                need = min(ws + bwin + pf - 2 - D, int(s["T1"][z - 2]))
                assert tq <= need, ((x, y, z), q)       # covered by the progress wait


@pytest.mark.parametrize("bwin,pf", WP)
@pytest.mark.parametrize("level", [3, 5, 7, 9])
def test_warps_own_one_row_at_a_time(level, bwin, pf):
    s = _lib.batch_schedule(level, bwin, pf)
    n = 2 ** level
    for z in range(1, n - 2):
        busy = {}
        for y in range(1, n - 1 - z):
            r = row_id(n, z, y)
            w, st, m = int(s["warp"][r]), int(s["start"][r]), n - 1 - z - y
            assert 0 <= w < 8
            assert st >= busy.get(w, -1), (z, y)
            busy[w] = st + m
            if y > 1:
                assert st >= int(s["start"][r - 1]) + bwin + 1 + pf


def _simulate(level, backward, bwin, pf):
    s, _, T0 = schedule(level, bwin, pf)
    n = 2 ** level
    nl = n - 3
    Tmax, D = s["Tmax"], s["D"]
    T1 = {z: int(s["T1"][z - 1]) for z in range(1, n - 2)}
    lo = {z: (Tmax - T1[z] if backward else T0[z]) for z in T1}
    hi = {z: (Tmax - T0[z] if backward else T1[z]) for z in T1}
    prog, pos, done = {z: -1 for z in T1}, dict(lo), set()
    order = range(nl, 0, -1) if backward else range(1, nl + 1)
    moved = True
    while moved:
        moved = False
        for z in order:
            if z in done:
                continue
            dep = z + 1 if backward else z - 1
            if dep in T1 and prog[dep] < min(pos[z] + bwin + pf - 2 - D, hi[dep]):
                continue
            t1 = min(pos[z] + bwin, hi[z] + 1)
            prog[z], pos[z], moved = t1 - 1, t1, True
            if t1 > hi[z]:
                done.add(z)
    return len(done) == nl


@pytest.mark.parametrize("bwin,pf", WP)
@pytest.mark.parametrize("level", [2, 3, 4, 5, 6, 7, 8])
def test_handoff_completes(level, bwin, pf):
    assert _simulate(level, backward=False, bwin=bwin, pf=pf)
    assert _simulate(level, backward=True, bwin=bwin, pf=pf)


UPPER_READS = [(1, 0, 0), (0, 1, 0), (-1, 1, 0), (1, -1, 1), (0, -1, 1), (0, 0, 1), (-1, 0, 1)]


@pytest.mark.parametrize("bwin,pf", WP)
@pytest.mark.parametrize("level", [2, 3, 4, 5, 6])
def test_backward_reads_are_safe(level, bwin, pf):
    """Backward = time reversal: point p runs at Tmax - T(p) and reads its upper neighbours."""
    s, T, T0 = schedule(level, bwin, pf)
    n = 2 ** level
    D, Tmax = s["D"], s["Tmax"]
    T1 = {z: int(s["T1"][z - 1]) for z in range(1, n - 2)}
    for (x, y, z), t in T.items():
        tb = Tmax - t
        m = n - 1 - z - y
        k = m - x                      # 0-based position along the descending row
        load_t = tb - k if k < pf else tb - pf
        ws = window_start(load_t, Tmax - T1[z], bwin)
        for dx, dy, dz in UPPER_READS:
            q = (x + dx, y + dy, z + dz)
            if q not in T:
                continue
            tq = Tmax - T[q]
            if dz == 0 and dy == 0:
                assert tq == tb - 1
            elif dz == 0:
                assert tq < ws, ((x, y, z), q)
            else:
                need = min(ws + bwin + pf - 2 - D, Tmax - T0[z + 1])
                assert tq <= need, ((x, y, z), q)

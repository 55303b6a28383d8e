"""numpy restatement of the reference's multigrid transfers and V-cycle on one all-Dirichlet
macro-tet -- TEST INFRASTRUCTURE ONLY (tests/ import it; the product never does).

Follows /root/reference/pkg/src/tetilu/multigrid.py: ``build_prolongation`` (:241-277, parity classes
``_PARITY_ENDPOINTS`` :230-238), ``Hierarchy.v_cycle`` (:459-485).  The products ``P.T @ r`` and
``P @ e`` are restated in scipy's accumulation order (csc: ascending fine index per coarse entry;
csr: ascending coarse index per fine entry), so they are bitwise the reference's; pinned by
tests/golden/mg_*.npz (generated from the live reference by tests/golden/make_mg.py).
"""

from __future__ import annotations

import numpy as np

PARITY_ENDPOINTS = {1: (-1, 0, 0), 2: (0, -1, 0), 4: (0, 0, -1), 3: (1, -1, 0), 5: (1, 0, -1),
                    6: (0, 1, -1), 7: (-1, 1, -1)}
# the 14 edge directions + centre in ascending (dz, dy, dx) order = ascending fine rank
OFFSETS_SORTED = sorted([(0, 0, 0)] + [s for a in PARITY_ENDPOINTS.values() for s in (a, tuple(-v for v in a))],
                        key=lambda o: (o[2], o[1], o[0]))


def _rank(c, n):
    c = np.asarray(c, dtype=np.int64)
    x, y, z = c[..., 0], c[..., 1], c[..., 2]
    zoff = (n + 1) * (n + 2) * (n + 3) // 6 - (n - z + 1) * (n - z + 2) * (n - z + 3) // 6
    return zoff + y * (n - z + 1) - y * (y - 1) // 2 + x


def _coords(n, interior):
    lo, out = (1, []) if interior else (0, [])
    for z in range(lo, n + 1):
        for y in range(lo, n + 1 - z):
            for x in range(lo, n + 1 - z - y):
                if not interior or x + y + z <= n - 1:
                    out.append((x, y, z))
    return np.array(out, dtype=np.int64).reshape(-1, 3)


def restrict(r_fine: np.ndarray, coarse_level: int) -> np.ndarray:
    """rc = P^T r on interior coarse points, 0 elsewhere."""
    nc = 2 ** coarse_level
    nf = 2 * nc
    C = _coords(nc, True)
    rc = np.zeros((nc + 1) * (nc + 2) * (nc + 3) // 6)
    acc = np.zeros(len(C))
    for off in OFFSETS_SORTED:
        v = r_fine[_rank(2 * C + np.array(off), nf)]
        acc = acc + (v if off == (0, 0, 0) else 0.5 * v)
    rc[_rank(C, nc)] = acc
    return rc


def prolong(e_coarse: np.ndarray, coarse_level: int) -> np.ndarray:
    """P e on interior fine points, 0 elsewhere."""
    nc = 2 ** coarse_level
    nf = 2 * nc
    F = _coords(nf, True)
    out = np.zeros((nf + 1) * (nf + 2) * (nf + 3) // 6)
    code = (F[:, 0] % 2) + 2 * (F[:, 1] % 2) + 4 * (F[:, 2] % 2)
    val = np.zeros(len(F))
    ev = code == 0
    val[ev] = e_coarse[_rank(F[ev] // 2, nc)]
    for c, a in PARITY_ENDPOINTS.items():
        sel = code == c
        half = (F[sel] + np.array(a)) // 2
        val[sel] = 0.5 * e_coarse[_rank(half, nc)] + 0.5 * e_coarse[_rank(half - np.array(a), nc)]
    out[_rank(F, nf)] = val
    return out

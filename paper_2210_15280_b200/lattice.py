"""Logical lattice of a refined macro-tetrahedron and its index conventions.

A macro-tet refined to level L carries micro-vertices at integer triples
(x, y, z) >= 0 with x + y + z <= n, n = 2**L.  Vectors are stored in full-lattice
rank order (z, then y, then x) -- the reference's API layout
(/root/reference/pkg/src/tetilu/geometry.py:120-215) that the drop-in boundary keeps.
The interior (x, y, z >= 1, x + y + z <= n - 1) carries the degrees of freedom.

Only what the smoother path needs lives here: direction tables, rank arithmetic,
the boundary band, and the macro-tet shapes the benchmark configurations use.
"""

from __future__ import annotations

import functools
from itertools import permutations

import numpy as np

# The 15 stencil directions and their lattice displacements (geometry.py:61-93).
DIRECTION_NAMES = ("w", "s", "se", "bnw", "bn", "bc", "be", "c",
                   "e", "n", "nw", "tse", "ts", "tc", "tw")
_DISP = {
    "w": (-1, 0, 0), "s": (0, -1, 0), "se": (1, -1, 0), "bnw": (-1, 1, -1), "bn": (0, 1, -1),
    "bc": (0, 0, -1), "be": (1, 0, -1), "c": (0, 0, 0),
}
_DISP.update({up: tuple(-v for v in _DISP[lo]) for lo, up in
              zip(("w", "s", "se", "bnw", "bn", "bc", "be"), ("e", "n", "nw", "tse", "ts", "tc", "tw"))})
OFFSETS = np.array([_DISP[name] for name in DIRECTION_NAMES], dtype=np.int64)
LOWER = tuple(range(7))          # directions preceding the centre in (z, y, x) order
UPPER = tuple(range(8, 15))
C = 7


def tet_points(m: int) -> int:
    """#{(x, y, z) >= 0 : x + y + z <= m}."""
    return 0 if m < 0 else (m + 1) * (m + 2) * (m + 3) // 6


def grid_size(level: int) -> int:
    return tet_points(2 ** level)


def interior_size(level: int) -> int:
    return tet_points(2 ** level - 4)


def rank_tables(level: int) -> np.ndarray:
    """rowoff[z, y] + x = full-lattice rank of (x, y, z); -1 outside the lattice."""
    n = 2 ** level
    z = np.arange(n + 1)[:, None]
    y = np.arange(n + 1)[None, :]
    zoff = tet_points(n) - (n - z + 1) * (n - z + 2) * (n - z + 3) // 6
    rowoff = zoff + y * (n - z + 1) - y * (y - 1) // 2
    return np.where(y <= n - z, rowoff, -1).astype(np.int64)


def lattice_rank(coords, level: int) -> np.ndarray:
    coords = np.atleast_2d(np.asarray(coords, dtype=np.int64))
    n = 2 ** level
    x, y, z = coords[:, 0], coords[:, 1], coords[:, 2]
    if np.any(coords < 0) or np.any(x + y + z > n):
        raise ValueError("coordinate outside the lattice")
    m = n - z
    return tet_points(n) - (m + 1) * (m + 2) * (m + 3) // 6 + y * (n - z + 1) - y * (y - 1) // 2 + x


@functools.lru_cache(maxsize=16)
def _lattice_coords_cached(level: int, region: str) -> np.ndarray:
    n = 2 ** level
    lo, top = (1, n - 1) if region == "interior" else (0, n)
    z, y = np.meshgrid(np.arange(lo, top + 1), np.arange(lo, top + 1), indexing="ij")
    z, y = z.ravel(), y.ravel()
    keep = top - z - y >= lo
    z, y = z[keep], y[keep]                       # rows in (z, y) lexicographic order
    cnt = top - z - y - lo + 1
    starts = np.cumsum(cnt) - cnt
    x = np.arange(int(cnt.sum())) - np.repeat(starts, cnt) + lo
    out = np.stack([x, np.repeat(y, cnt), np.repeat(z, cnt)], axis=1).astype(np.int64)
    out.setflags(write=False)
    return out


def lattice_coords(level: int, region: str = "full") -> np.ndarray:
    """Coordinates of the full lattice or its interior, in rank order, shape (N, 3) (read-only)."""
    if region not in ("full", "interior"):
        raise ValueError(f"unknown region {region!r}")
    return _lattice_coords_cached(int(level), region)


def is_interior(coords, level: int) -> np.ndarray:
    coords = np.atleast_2d(np.asarray(coords, dtype=np.int64))
    return (coords >= 1).all(axis=1) & (coords.sum(axis=1) < 2 ** level)


def interior_mask(level: int) -> np.ndarray:
    """Boolean mask over the full lattice (rank order) of interior points."""
    return is_interior(lattice_coords(level), level)


def band_mask(coords, level: int) -> np.ndarray:
    """Boundary band: interior points whose stencil reaches the boundary (surrogate.py:223-229)."""
    n = 2 ** level
    return (coords == 1).any(axis=1) | (coords.sum(axis=1) == n - 1)


def band_ranks(level: int) -> np.ndarray:
    inner = lattice_coords(level, "interior")
    return lattice_rank(inner[band_mask(inner, level)], level)


# ------------------------------------------------------------------------------------------
# macro-tet shapes used by the benchmark configurations (BASELINE.json "configs")
# ------------------------------------------------------------------------------------------

def unit_tet() -> np.ndarray:
    """(0,0,0), (1,0,0), (0,1,0), (0,0,1): configs 1 and 3 (reference trirect_tet(1.0))."""
    return np.array([(0.0, 0.0, 0.0), (1.0, 0.0, 0.0), (0.0, 1.0, 0.0), (0.0, 0.0, 1.0)])


def distorted_tet() -> np.ndarray:
    """Affinely distorted tet of configs 2 and 5."""
    return np.array([(0.0, 0.0, 0.0), (1.0, 0.1, 0.0), (0.2, 1.0, 0.0), (0.1, 0.3, 0.8)])


def kuhn_tet(path, origin=(0.0, 0.0, 0.0), size: float = 1.0) -> np.ndarray:
    """Kuhn simplex of a cube: walk from the origin corner along the axes in ``path``
    (the cube_mesh construction, geometry.py:537-570)."""
    p = np.array(origin, dtype=float)
    verts = [p.copy()]
    for axis in path:
        p = p.copy()
        p[axis] += size
        verts.append(p)
    return np.array(verts)


def kuhn_mesh(cells_per_axis: int = 4) -> list[np.ndarray]:
    """Config 4: a cells^3 array of unit cubes, each split into 6 Kuhn macro-tets,
    ordered (cube z, y, x, then path in lexicographic permutation order)."""
    tets = []
    for cz in range(cells_per_axis):
        for cy in range(cells_per_axis):
            for cx in range(cells_per_axis):
                for path in permutations(range(3)):
                    tets.append(kuhn_tet(path, (float(cx), float(cy), float(cz))))
    return tets

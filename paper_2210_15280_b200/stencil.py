"""Operator input of the smoother: 15-point P1 stiffness stencils on one macro-tet.

Host-side setup (runs once per macro-tet).  ``stencil_source`` returns the
operator the residual r = f - A u of every sweep uses, either one
translation-invariant row (constant coefficient: configs 1, 4) or one row per
lattice point (variable / tensor coefficient: configs 2, 3, 5).

The numerics restate the reference's assembly (reference assembly.py:46-221)
with the same numpy primitives on arrays of the same shape, so the rows are
bitwise identical to the reference's (pinned by tests/test_setup_parity.py);
the factorization and the least-squares fit downstream are sensitive to the last
ulp of these rows.
"""

from __future__ import annotations

import functools
from dataclasses import dataclass

import numpy as np

from . import lattice

# Six translation classes of the structured subdivision of a refined tet: vertex offsets
# from the class anchor.  Every edge lies along a stencil direction, which keeps the vertex
# neighbourhood 15-point.  Class / vertex order fixes the accumulation order of the rows.
ELEMENT_CLASSES = np.array(
    [
        [(0, 0, 0), (0, 0, 1), (0, 1, 0), (1, 0, 0)],
        [(0, 0, 1), (0, 1, 0), (0, 1, 1), (1, 0, 1)],
        [(0, 0, 1), (0, 1, 0), (1, 0, 0), (1, 0, 1)],
        [(0, 1, 0), (0, 1, 1), (1, 0, 1), (1, 1, 0)],
        [(0, 1, 0), (1, 0, 0), (1, 0, 1), (1, 1, 0)],
        [(0, 1, 1), (1, 0, 1), (1, 1, 0), (1, 1, 1)],
    ],
    dtype=np.int64,
)
_DIR_OF = {tuple(o): i for i, o in enumerate(lattice.OFFSETS)}


def _vertex_patch():
    """The 24 micro-elements around a vertex p: (class, local index of p, vertex offsets
    relative to p, stencil direction of each element vertex as seen from p)."""
    patch = []
    for ci in range(6):
        for li in range(4):
            rel = ELEMENT_CLASSES[ci] - ELEMENT_CLASSES[ci, li]
            dirs = [lattice.C if j == li else _DIR_OF[tuple(rel[j])] for j in range(4)]
            patch.append((ci, li, rel, dirs))
    return patch


VERTEX_PATCH = _vertex_patch()


class CoefficientField:
    """Diffusion coefficient K(x): constant scalar, scalar field or tensor field."""

    def __init__(self, fn=None, constant: float | None = None, name: str = ""):
        if (fn is None) == (constant is None):
            raise ValueError("pass exactly one of fn or constant")
        self.fn = fn
        self.const = None if constant is None else float(constant)
        self.name = name or ("constant" if fn is None else "field")

    @classmethod
    def constant(cls, value: float = 1.0) -> "CoefficientField":
        return cls(constant=value, name=f"constant({value:g})")

    @classmethod
    def scalar(cls, fn, name: str = "scalar") -> "CoefficientField":
        return cls(fn=lambda pts: np.asarray(fn(pts), dtype=np.float64), name=name)

    @classmethod
    def tensor(cls, fn, name: str = "tensor") -> "CoefficientField":
        return cls(fn=fn, name=name)

    @property
    def is_constant(self) -> bool:
        return self.const is not None

    def evaluate(self, points: np.ndarray) -> np.ndarray:
        """K at the points, shape (m, 3, 3)."""
        points = np.atleast_2d(points)
        m = len(points)
        if self.const is not None:
            return np.broadcast_to(self.const * np.eye(3), (m, 3, 3))
        vals = np.asarray(self.fn(points), dtype=np.float64)
        if vals.shape == (m,):
            return vals[:, None, None] * np.eye(3)
        if vals.shape == (m, 3, 3):
            return vals
        raise ValueError("coefficient function must return (m,) or (m, 3, 3)")


def element_matrices(verts: np.ndarray, K: np.ndarray) -> np.ndarray:
    """P1 stiffness |T| grad(phi_i)^T K grad(phi_j) of a batch of tets (m, 4, 3) with
    one-point quadrature K (m, 3, 3) -> (m, 4, 4)."""
    verts = np.asarray(verts, dtype=np.float64)
    E = verts[:, 1:] - verts[:, :1]
    det = np.linalg.det(E)
    scale = np.linalg.norm(E, axis=2).max(axis=1)
    if np.any(np.abs(det) <= 1e-14 * scale ** 3):
        raise ValueError("degenerate micro-element")
    grads = np.empty((len(verts), 4, 3))
    grads[:, 1:] = np.linalg.inv(E).transpose(0, 2, 1)
    grads[:, 0] = -grads[:, 1:].sum(axis=1)
    return np.einsum("m,mid,mde,mje->mij", np.abs(det) / 6.0, grads, K, grads, optimize=True)


@functools.lru_cache(maxsize=8)
def _float_coords(level: int) -> np.ndarray:
    out = lattice.lattice_coords(level).astype(np.float64)
    out.setflags(write=False)
    return out


def micro_positions(vertices: np.ndarray, level: int) -> np.ndarray:
    """Physical position of every lattice point (rank order): v0 + (x d1 + y d2 + z d3) / n."""
    v = np.asarray(vertices, dtype=np.float64)
    return v[0] + _float_coords(level) @ (v[1:] - v[0]) / 2 ** level


@dataclass
class StencilSource:
    """Operator rows of one refined macro-tet: ``data`` is one row (constant) or
    [grid_size, 15] with only interior rows filled (reference assembly.py:173-194)."""

    level: int
    data: np.ndarray
    constant: bool

    @property
    def kernel_args(self) -> tuple[np.ndarray, bool]:
        return np.atleast_2d(self.data), self.constant

    def row(self, p) -> np.ndarray:
        if self.constant:
            return self.data.copy()
        return self.data[int(lattice.lattice_rank(np.asarray(p)[None], self.level)[0])].copy()


def _deep_point(level: int) -> np.ndarray:
    q = max(1, 2 ** level // 4)
    return np.array((q, q, q), dtype=np.int64)


def stencil_source(vertices, level: int, coeff: CoefficientField) -> StencilSource:
    """Assemble the 15-point rows of the P1 operator -div(K grad u) on a refined macro-tet."""
    vertices = np.asarray(getattr(vertices, "vertices", vertices), dtype=np.float64)
    pos = micro_positions(vertices, level)
    if coeff.is_constant:
        p = _deep_point(level)
        row = np.zeros(15)
        for ci, li, rel, dirs in VERTEX_PATCH:
            verts = pos[lattice.lattice_rank(p + rel, level)]
            S = element_matrices(verts[None], coeff.evaluate(verts.mean(axis=0)[None]))[0]
            for j in range(4):
                row[dirs[j]] += S[li, j]
        return StencilSource(level, row, True)

    inner = lattice.lattice_coords(level, "interior")
    iranks = lattice.lattice_rank(inner, level)
    data = np.zeros((lattice.grid_size(level), 15))
    for ci, li, rel, dirs in VERTEX_PATCH:
        ranks = lattice.lattice_rank((inner[:, None, :] + rel[None]).reshape(-1, 3), level).reshape(-1, 4)
        verts = pos[ranks]
        S = element_matrices(verts, coeff.evaluate(verts.mean(axis=1)))
        for j in range(4):
            data[iranks, dirs[j]] += S[:, li, j]
    return StencilSource(level, data, False)


def sin_kappa() -> CoefficientField:
    """Config 3's coefficient k(x) = 1 + 0.5 sin(2 pi x) sin(2 pi y) sin(2 pi z)."""
    def fn(p):
        p = np.atleast_2d(p)
        return 1.0 + 0.5 * np.sin(2 * np.pi * p[:, 0]) * np.sin(2 * np.pi * p[:, 1]) * np.sin(2 * np.pi * p[:, 2])
    return CoefficientField.scalar(fn, name="sin_kappa")


def diag_tensor(diag) -> CoefficientField:
    """Constant anisotropic tensor K = diag(...) given as a field (configs 2, 5)."""
    d = np.diag(np.asarray(diag, dtype=np.float64))
    return CoefficientField.tensor(lambda pts: np.broadcast_to(d, (len(np.atleast_2d(pts)), 3, 3)),
                                   name=f"diag{tuple(diag)}")

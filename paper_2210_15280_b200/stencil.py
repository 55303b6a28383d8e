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
class SeparableK:
    """Table form of a separable scalar coefficient's rows on the unit macro-tet: k at a centroid
    (4p + a) / (4n) is c0 + (tables[0][4x+ax] * tables[1][4y+ay]) * tables[2][4z+az]; the rows
    follow from separable_program (compiled into csrc/tilu_sepk.h).  W = n^2 |T|."""

    level: int
    tables: np.ndarray   # [3][4n+1]
    c0: float
    w: float

    def rows(self) -> np.ndarray:
        """[grid][15] rows (interior filled, zero elsewhere) from the native builder."""
        import ctypes

        from . import _lib
        out = np.zeros((lattice.grid_size(self.level), 15))
        tab = np.ascontiguousarray(self.tables, dtype=np.float64)
        _lib.check(_lib.lib().tilu_sepk_rows(self.level, tab.ctypes.data, ctypes.c_double(self.c0),
                                             ctypes.c_double(self.w), out.ctypes.data))
        return out


@dataclass
class StencilSource:
    """Operator rows of one refined macro-tet: ``data`` is one row (constant) or
    [grid_size, 15] with only interior rows filled (reference assembly.py:173-194)."""

    level: int
    data: np.ndarray
    constant: bool
    sepk: "SeparableK | None" = None   # table form of the rows (separable coefficient, unit tet)

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


def stencil_source(vertices, level: int, coeff: CoefficientField, *, native: bool = True) -> StencilSource:
    """Assemble the 15-point rows of the P1 operator -div(K grad u) on a refined macro-tet.

    A separable scalar coefficient on the unit macro-tet (config 3) is assembled by the native
    row builder (``tilu_sepk_rows``: the same rows bitwise, in seconds instead of the numpy path's
    ~30 min at level 9), and the source keeps the table form (``sepk``) so the GPU residual can
    evaluate the rows on the fly instead of reading them; ``native=False`` forces the numpy path."""
    vertices = np.asarray(getattr(vertices, "vertices", vertices), dtype=np.float64)
    if isinstance(coeff, SeparableScalar) and separable_program(vertices, level) is not None:
        sk = SeparableK(level, coeff.tables(level), coeff.c0, separable_program(vertices, level)[1])
        if native:
            return StencilSource(level, sk.rows(), False, sk)
        src = stencil_source(vertices, level, CoefficientField.scalar(coeff.fn, coeff.name), native=False)
        return StencilSource(level, src.data, False, sk)
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


class SeparableScalar(CoefficientField):
    """Scalar coefficient k(x, y, z) = c0 + c1 * gx(x) * gy(y) * gz(z), evaluated left to right in
    exactly that order (so its values are bitwise those of the same Python expression).  Besides
    the generic per-point assembly, a separable field on the unit macro-tet has a table form
    (``tables``) that the native row builder and the GPU residual evaluate on the fly."""

    def __init__(self, gx, gy, gz, c0: float = 0.0, c1: float = 1.0, name: str = "separable"):
        self.gx, self.gy, self.gz = gx, gy, gz
        self.c0, self.c1 = float(c0), float(c1)

        def fn(p):
            p = np.atleast_2d(p)
            return self.c0 + self.c1 * gx(p[:, 0]) * gy(p[:, 1]) * gz(p[:, 2])
        super().__init__(fn=lambda pts: np.asarray(fn(pts), dtype=np.float64), name=name)

    def tables(self, level: int) -> np.ndarray:
        """[3][4n+1]: c1*gx, gy, gz at the abscissae c / (4n), c = 0..4n -- every coordinate a
        micro-element centroid of the unit macro-tet can take (the mean of four lattice points)."""
        n = 2 ** level
        t = np.arange(4 * n + 1, dtype=np.float64) / (4.0 * n)
        return np.ascontiguousarray(np.stack([self.c1 * self.gx(t), self.gy(t), self.gz(t)]), dtype=np.float64)


def _sin2pi(t):
    return np.sin(2 * np.pi * t)


def sin_kappa() -> SeparableScalar:
    """Config 3's coefficient k(x) = 1 + 0.5 sin(2 pi x) sin(2 pi y) sin(2 pi z)."""
    return SeparableScalar(_sin2pi, _sin2pi, _sin2pi, c0=1.0, c1=0.5, name="sin_kappa")


# ------------------------------------------------------------------------------------------
# on-the-fly rows of a separable scalar coefficient on the unit macro-tet
# ------------------------------------------------------------------------------------------

def separable_program(vertices, level: int):
    """The per-point rows of a scalar coefficient as a fixed program, or None if the macro-tet does
    not admit it.

    On the unit macro-tet every micro-element has gradients in {0, +-n} and the same volume, so
    element_matrices' einsum (path: K contracted with grads, then with grads, then the volume)
    reduces, for K = k I, to  S[li, j] = fl(fl(m k) W)  with the integer m = sum_e g_li,e g_j,e / n^2
    in {-2..3} and W = n^2 |T| (exact power-of-two scaling), and the element's centroid is exactly
    (4p + a) / (4n) for a small integer offset a.  Row entry d of point p is the sum of those
    contributions over the 24 elements of VERTEX_PATCH in patch order (zero contributions dropped:
    adding +-0 to the +0-initialised accumulator is the identity).
    Returns (elements, W): elements[e] = ((ax, ay, az), [(direction, m), ...]) in patch order."""
    vertices = np.asarray(getattr(vertices, "vertices", vertices), dtype=np.float64)
    if not np.array_equal(vertices, lattice.unit_tet()):
        return None
    n = 2 ** level
    pos = micro_positions(vertices, level)
    p = _deep_point(level)
    elements, vols = [], set()
    for ci, li, rel, dirs in VERTEX_PATCH:
        verts = pos[lattice.lattice_rank(p + rel, level)][None]
        E = verts[:, 1:] - verts[:, :1]
        det = np.linalg.det(E)
        g = np.empty((1, 4, 3))
        g[:, 1:] = np.linalg.inv(E).transpose(0, 2, 1)
        g[:, 0] = -g[:, 1:].sum(axis=1)
        g = g[0] / n
        if not np.all(np.isin(g, (-1.0, 0.0, 1.0))):
            return None
        vols.add(float(np.abs(det[0]) / 6.0))
        contrib = []
        for j in range(4):
            m = int(sum(g[li, e] * g[j, e] for e in range(3)))
            if m != 0:
                contrib.append((int(dirs[j]), m))
        elements.append((tuple(int(v) for v in rel.sum(axis=0)), contrib))
    if len(vols) != 1:
        return None
    return elements, vols.pop() * float(n) ** 2


def diag_tensor(diag) -> CoefficientField:
    """Constant anisotropic tensor K = diag(...) given as a field (configs 2, 5)."""
    d = np.diag(np.asarray(diag, dtype=np.float64))
    return CoefficientField.tensor(lambda pts: np.broadcast_to(d, (len(np.atleast_2d(pts)), 3, 3)),
                                   name=f"diag{tuple(diag)}")

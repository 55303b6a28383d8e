"""CPU checks of the 8(f) rows' host side: the numpy restatement of the multigrid transfers is pinned
bitwise by the reference's golden vectors (tests/golden/mg_*.npz, from the live reference), the level
schedule of the CSR block solves is a valid topological schedule, and the coarsest-level matrix built
from stencil rows is the operator's interior block."""
import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import mg_oracle as MO
from paper_2210_15280_b200 import _lib, lattice
from paper_2210_15280_b200 import stencil as S


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "mg_*.npz"))))
def test_transfer_restatement_pinned_by_reference(path):
    d = np.load(path)
    cl = int(d["lmax"]) - 1
    assert np.array_equal(MO.restrict(d["xfer_r"], cl), d["xfer_rc"])
    assert np.array_equal(MO.prolong(d["xfer_e"], cl), d["xfer_pe"])


def test_restriction_is_transpose_of_prolongation():
    cl = 3
    rng = np.random.default_rng(0)
    r = np.where(lattice.interior_mask(cl + 1), rng.standard_normal(lattice.grid_size(cl + 1)), 0.0)
    e = np.where(lattice.interior_mask(cl), rng.standard_normal(lattice.grid_size(cl)), 0.0)
    assert abs(MO.restrict(r, cl) @ e - r @ MO.prolong(e, cl)) <= 1e-12 * abs(r @ MO.prolong(e, cl))


def test_csr_levels_schedule():
    import ctypes

    sparse = pytest.importorskip("scipy.sparse")
    rng = np.random.default_rng(1)
    m = 200
    A = sparse.random(m, m, 0.03, random_state=2, format="csr") + sparse.identity(m, format="csr")
    A = (A + A.T).tocsr()
    A.sort_indices()
    indptr, indices = A.indptr.astype(np.int64), A.indices.astype(np.int32)
    for upper in (0, 1):
        level = np.zeros(m, dtype=np.int32)
        nl = _lib.lib().tilu_csr_levels(m, indptr.ctypes.data, indices.ctypes.data, upper, level.ctypes.data)
        assert nl == level.max() + 1
        for i in range(m):
            deps = [j for j in indices[indptr[i]:indptr[i + 1]] if (j > i if upper else j < i)]
            assert all(level[j] < level[i] for j in deps)
            assert level[i] == (max(level[j] for j in deps) + 1 if deps else 0)
    assert rng is not None
    assert _lib.lib().tilu_csr_levels(-1, None, None, 0, None) == -1


def test_coarse_matrix_from_stencil_rows():
    from paper_2210_15280_b200.multigrid import interior_matrix

    src = S.stencil_source(lattice.distorted_tet(), 3, S.diag_tensor((1, 1, 1e-1)))
    A = interior_matrix(src)
    assert A.shape == (35, 35)
    assert np.allclose(A, A.T, rtol=1e-12, atol=1e-14) and np.all(np.linalg.eigvalsh(0.5 * (A + A.T)) > 0)
    # a row of the matrix applied to a vector equals the stencil applied at that point
    u = np.zeros(lattice.grid_size(3))
    inner = lattice.lattice_coords(3, "interior")
    ranks = lattice.lattice_rank(inner, 3)
    u[ranks] = np.random.default_rng(3).standard_normal(35)
    p = inner[17]
    row = src.data[ranks[17]]
    want = sum(row[d] * u[lattice.lattice_rank((p + lattice.OFFSETS[d])[None], 3)[0]] for d in range(15))
    assert abs(A[17] @ u[ranks] - want) <= 1e-13 * max(1.0, abs(want))

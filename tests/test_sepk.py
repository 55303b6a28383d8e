"""Config 3's separable coefficient rows (stencil.SeparableK, csrc/tilu_sepk.h) -- CPU.

The on-the-fly program must reproduce the reference's per-point assembly (assembly.py:208-221,
element_stiffness_batch :102-123) bitwise: against the reference's own rows (golden cfg3 fixtures,
generated from the live reference) and against this repo's numpy restatement of the assembly."""
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import GOLDEN, ROOT
from paper_2210_15280_b200 import lattice
from paper_2210_15280_b200 import stencil as S


def test_generated_program_is_up_to_date():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "gen_sepk.py"), "--check"], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("level", [4, 5])
def test_native_rows_equal_reference_rows(level):
    g = np.load(os.path.join(GOLDEN, f"cfg3_L{level}_v1.npz"))
    src = S.stencil_source(lattice.unit_tet(), level, S.sin_kappa())
    assert src.sepk is not None
    mask = lattice.interior_mask(level)
    assert np.array_equal(src.data[mask], g["arows"][mask])


@pytest.mark.parametrize("level", [3, 4, 5, 6])
def test_native_rows_equal_numpy_assembly(level):
    a = S.stencil_source(lattice.unit_tet(), level, S.sin_kappa())
    b = S.stencil_source(lattice.unit_tet(), level, S.sin_kappa(), native=False)
    assert np.array_equal(a.data, b.data)
    assert b.sepk is not None and a.sepk.w == b.sepk.w


def test_separable_field_values_equal_the_config3_expression():
    pts = np.random.default_rng(0).uniform(0, 1, (1000, 3))
    want = 1.0 + 0.5 * np.sin(2 * np.pi * pts[:, 0]) * np.sin(2 * np.pi * pts[:, 1]) * np.sin(2 * np.pi * pts[:, 2])
    got = S.sin_kappa().evaluate(pts)[:, 0, 0]
    assert np.array_equal(got, want)


def test_program_only_for_the_unit_tet():
    assert S.separable_program(lattice.distorted_tet(), 5) is None
    assert S.separable_program(lattice.kuhn_tet((1, 0, 2)), 5) is None
    el, w = S.separable_program(lattice.unit_tet(), 6)
    assert len(el) == 24 and w > 0
    # a non-unit tet with a separable field takes the generic per-point path (no table form)
    src = S.stencil_source(lattice.distorted_tet(), 3, S.sin_kappa())
    assert src.sepk is None and not src.constant


def test_tables_cover_every_centroid():
    t = S.sin_kappa().tables(5)
    assert t.shape == (3, 4 * 32 + 1)
    c = np.arange(4 * 32 + 1) / 128.0
    assert np.array_equal(t[1], np.sin(2 * np.pi * c))
    assert np.array_equal(t[0], 0.5 * np.sin(2 * np.pi * c))

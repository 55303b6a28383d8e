"""Config 3 at full size (level 9) -- the fixture that pins the GPU sweep at the north star's level.

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_config3_l9.py     # ~15 min, ~12 GB RAM

Setup (this repo's host setup, whose arrays are bitwise the reference's at levels 4-5:
tests/test_setup_parity.py, tests/test_sepk.py): unit macro-tet, level 9, k(x) = 1 + 0.5 sin(2 pi x)
sin(2 pi y) sin(2 pi z) (per-point rows from the native builder == the reference's stencil_source
rows), q = 6 -> build_surrogate_ilu with single-threaded BLAS.  Inputs as BASELINE.json configs[2]:
f ~ N(0, 1) (numpy default_rng(3), interior rank order), u = 0, 100 sweeps.  The C oracle
(oracle/tilu_oracle.c, the reference kernels' bitwise restatement) runs the sweeps.

Stored (tests/golden/l9_config3.npz, small): the fitted arrays (lcoefs, dcoefs; the LSQ depends on the
host BLAS, so the GPU test uses these instead of refitting), the coefficient tables, W, SHA-256 of
the band rows (recomputed by the deterministic native factorization on the GPU box and checked),
the per-sweep residual norms ||f - A u_k||^2 (k = 0..99, before each sweep) and after the last sweep,
SHA-256 of the full u after sweeps 1, 2, 3 and 100, and u at every 1999th interior point after
those sweeps.  The 2.7 GB rows and the 181 MB vectors are not stored.
"""
from __future__ import annotations

import hashlib
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2210_15280_b200 import fitting, lattice, stencil  # noqa: E402

LEVEL, Q, SWEEPS, FSEED, STEP = 9, 6, 100, 3, 1999
SNAP = (1, 2, 3, 100)
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "l9_config3.npz")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def inputs(level: int = LEVEL):
    mask = lattice.interior_mask(level)
    f = np.zeros(lattice.grid_size(level))
    f[mask] = np.random.default_rng(FSEED).normal(size=int(mask.sum()))
    return f, np.zeros_like(f)


def main():
    t0 = time.time()
    src = stencil.stencil_source(lattice.unit_tet(), LEVEL, stencil.sin_kappa())
    print(f"rows {time.time() - t0:.1f}s", flush=True)
    fit = fitting.fit_surrogate_ilu(src, LEVEL, (Q, Q, Q), "v1")
    print(f"fit {time.time() - t0:.1f}s eff {fit.degrees} stride {fit.stride}", flush=True)
    f, u = inputs()
    iranks = lattice.lattice_rank(lattice.lattice_coords(LEVEL, "interior"), LEVEL)
    sample = iranks[::STEP]
    sur = O.OracleSurrogate(LEVEL, fit.lcoefs, fit.dcoefs, "v1", fit.band_ranks, fit.store_rows)
    norms, hashes, snaps = [], {}, {}
    for k in range(1, SWEEPS + 1):
        norms.append(float(O.sweeps(sur, LEVEL, src.data, u, f, 1, return_norms=True)[0]))
        if k in SNAP:
            hashes[k] = sha(u)
            snaps[k] = u[sample].copy()
            print(f"sweep {k} {time.time() - t0:.1f}s rnorm2 {norms[-1]:.6e}", flush=True)
    r = f - O.stencil_apply(LEVEL, src.data, u)
    mask = lattice.interior_mask(LEVEL)
    final = float(np.sum(r[mask] ** 2))
    np.savez_compressed(
        OUT, level=LEVEL, q=Q, sweeps=SWEEPS, fseed=FSEED, step=STEP, snaps=np.array(SNAP),
        lcoefs=fit.lcoefs, dcoefs=fit.dcoefs, eff_degrees=np.array(fit.degrees), stride=fit.stride,
        tables=src.sepk.tables, c0=src.sepk.c0, w=src.sepk.w,
        band_sha=sha(fit.store_rows), band_ranks_sha=sha(fit.band_ranks), rows_sha=sha(src.data),
        rnorm2=np.array(norms), rnorm2_final=final,
        u_sha=np.array([hashes[k] for k in SNAP]), u_sample=np.stack([snaps[k] for k in SNAP]),
        sample_ranks=sample)
    print(f"wrote {OUT} ({os.path.getsize(OUT) / 1e3:.0f} kB) in {time.time() - t0:.0f}s")


if __name__ == "__main__":
    main()

"""Config 3 at level 9 swept by the REFERENCE's own Numba kernels (build container only): r = f - A u
(_kernels.stencil_apply), SurrogateILU.solve_into (surrogate_forward / surrogate_backward), u += w
(multigrid.py:414-429), on this repo's setup arrays -- which tests/golden/fit_cfg3_L9_ref.npz proves bit-identical
to the reference's own setup.  Stores SHA-256 of the full iterate after sweeps 1, 2, 3 (and 100 with --full, ~20
min) -> tests/golden/l9_reference_sweeps.npz; tests/test_oracle_golden.py compares them with l9_config3.npz, the
C oracle's run that the GPU parity test and the bench are pinned to.

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_l9_reference_sweeps.py [--full]
"""
import hashlib
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
import numpy as np  # noqa: E402

from tetilu import _kernels, geometry  # noqa: E402  (the unmodified reference)

from paper_2210_15280_b200 import fitting, lattice, stencil  # noqa: E402
from make_config3_l9 import FSEED, LEVEL, Q, inputs, sha  # noqa: E402

if __name__ == "__main__":
    snaps = (1, 2, 3, 100) if "--full" in sys.argv else (1, 2, 3)
    t0 = time.time()
    src = stencil.stencil_source(lattice.unit_tet(), LEVEL, stencil.sin_kappa())
    fit = fitting.fit_surrogate_ilu(src, LEVEL, (Q, Q, Q), "v1")
    print(f"setup {time.time() - t0:.0f}s", flush=True)
    n = 2 ** LEVEL
    _, rowoff = geometry.rank_tables(LEVEL)
    lcoefs, dcoefs = np.ascontiguousarray(fit.lcoefs), np.ascontiguousarray(fit.dcoefs)
    band, store = np.ascontiguousarray(fit.band_ranks), np.ascontiguousarray(fit.store_rows)
    f, u = inputs()
    mask = lattice.interior_mask(LEVEL)
    out, w = np.zeros_like(u), np.zeros_like(u)
    hashes = {}
    for k in range(1, max(snaps) + 1):
        _kernels.stencil_apply(n, rowoff, src.data, False, u, out)
        w[:] = 0.0
        w[mask] = f[mask] - out[mask]
        _kernels.surrogate_forward(n, rowoff, 1.0 / n, lcoefs, w, True, band, store)
        _kernels.surrogate_backward(n, rowoff, 1.0 / n, lcoefs, dcoefs, w, True, band, store)
        u[mask] += w[mask]
        if k in snaps:
            hashes[k] = sha(u)
            print(f"sweep {k} {time.time() - t0:.0f}s {hashes[k][:16]}", flush=True)
    np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "l9_reference_sweeps.npz"),
                        snaps=np.array(snaps), u_sha=np.array([hashes[k] for k in snaps]), level=LEVEL, q=Q, fseed=FSEED)
    print("done", time.time() - t0)

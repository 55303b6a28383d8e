"""Config 3's setup with the UNMODIFIED reference at the north star's size (build container only; ~30 min,
~28 GB): stencil_source (level 9, k = 1 + 0.5 sin sin sin) and build_surrogate_ilu(q = 6).  Stores the fitted
arrays in full and SHA-256 of the per-point rows, band ranks and band store -> tests/golden/fit_cfg3_L9_ref.npz,
which tests/test_setup_parity.py compares with the arrays of l9_config3.npz (this repo's setup).

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_fit_l9_reference.py
"""
import hashlib
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")
import numpy as np  # noqa: E402

sys.path.insert(0, "/root/reference/pkg/src")
OUT = os.path.dirname(os.path.abspath(__file__))
from tetilu import geometry  # noqa: E402
from tetilu.assembly import CoefficientField, stencil_source  # noqa: E402
from tetilu.surrogate import build_surrogate_ilu  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def kappa(p):
    p = np.atleast_2d(p)
    return 1.0 + 0.5 * np.sin(2 * np.pi * p[:, 0]) * np.sin(2 * np.pi * p[:, 1]) * np.sin(2 * np.pi * p[:, 2])


if __name__ == "__main__":
    level, q = 9, 6
    t = time.time()
    src = stencil_source(geometry.MacroTet(geometry.trirect_tet(1.0)), level, CoefficientField.scalar(kappa))
    t_rows = time.time() - t
    rows_sha = sha(src.data)
    t = time.time()
    sur = build_surrogate_ilu(src, level, (q, q, q), variant="v1")
    t_fit = time.time() - t
    np.savez_compressed(os.path.join(OUT, "fit_cfg3_L9_ref.npz"), level=level, q=q, lcoefs=sur._lcoefs, dcoefs=sur._dcoefs,
                        eff_degrees=np.array(sur.degrees), stride=sur.stride, rows_sha=rows_sha,
                        band_sha=sha(sur._band_ranks), store_sha=sha(sur._store_rows), nband=len(sur._band_ranks),
                        stencil_source_s=t_rows, build_s=t_fit)
    print("done", sur.degrees, sur.stride, t_rows, t_fit)

"""Setup parity (P2) at the benchmark levels: the UNMODIFIED reference's build_surrogate_ilu (build container only)
for config 4's Kuhn macro-tet at level 7 (q = 6) and config 5's distorted tet at level 8 (q = 4) -- the fitted
arrays in full, the V1 band store as a SHA-256 (2-9 MB otherwise).  -> tests/golden/fit_*.npz

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_fit_large.py
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


def case(name, verts, coeff, level, q):
    t = time.time()
    src = stencil_source(geometry.MacroTet(np.asarray(verts, dtype=float)), level, coeff)
    sur = build_surrogate_ilu(src, level, (q, q, q), variant="v1")
    np.savez_compressed(os.path.join(OUT, name + ".npz"), verts=np.asarray(verts, dtype=float), level=level, q=q,
                        lcoefs=sur._lcoefs, dcoefs=sur._dcoefs, eff_degrees=np.array(sur.degrees), stride=sur.stride,
                        band_sha=sha(sur._band_ranks), store_sha=sha(sur._store_rows), nband=len(sur._band_ranks))
    print(name, sur.degrees, sur.stride, f"{time.time() - t:.1f}s")


if __name__ == "__main__":
    kuhn = [(0, 0, 0), (1, 0, 0), (1, 1, 0), (1, 1, 1)]
    case("fit_kuhn_L7_q6", kuhn, CoefficientField.constant(1.0), 7, 6)
    diag = np.diag([1.0, 1e-2, 1.0])
    case("fit_cfg5_L8_q4", [(0, 0, 0), (1, 0.1, 0), (0.2, 1, 0), (0.1, 0.3, 0.8)],
         CoefficientField.tensor(lambda p: np.broadcast_to(diag, (len(np.atleast_2d(p)), 3, 3))), 8, 4)

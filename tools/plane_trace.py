"""Per-task timeline of the plane kernels (TILU_PLANE_TRACE=<file> run of tools/plane_bench.py):
band lag (start of (b, c) after (b-1, c)), chunk lag (after (b, c-1)), task duration and the
implied step time, for the forward (pass 0) and backward (pass 1) kernels.
    python tools/plane_trace.py <trace file> <level>"""
import sys

import numpy as np

path, level = sys.argv[1], int(sys.argv[2])
n = 2 ** level
rows = [l.split() for l in open(path) if l[0].isdigit()]
for pas in (0, 1):
    R = [r for r in rows if int(r[0]) == pas]
    st, en = {}, {}
    for r in R:
        b, c = int(r[2]), int(r[3])
        st[(b, c)], en[(b, c)] = int(r[4]), int(r[5])
    t0 = min(st.values())
    dur, steps, blag, clag = [], [], [], []
    for (b, c), s in st.items():
        s0, z0 = 2 + 4 * b, 1 + 32 * c
        T = (z0 + 32 + n - 1 - s0) - (z0 - 3) + 1
        dur.append(en[(b, c)] - s)
        steps.append((en[(b, c)] - s) / T)
        nb = (b + 1, c) if pas == 1 else (b - 1, c)
        if nb in st:
            blag.append(s - st[nb])
        nc = (b, c + 1) if pas == 1 else (b, c - 1)
        if nc in st:
            clag.append(s - st[nc])
    span = max(en.values()) - t0
    print(f"pass {pas}: {len(st)} tasks, span {span / 1e3:.1f} us; step ns median {np.median(steps):.0f} "
          f"p10 {np.percentile(steps, 10):.0f} p90 {np.percentile(steps, 90):.0f}; band lag us median "
          f"{np.median(blag) / 1e3:.2f} p90 {np.percentile(blag, 90) / 1e3:.2f}; chunk lag us median "
          f"{np.median(clag) / 1e3:.2f}; task us median {np.median(dur) / 1e3:.1f}")

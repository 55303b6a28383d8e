"""Run one traced packed sweep (TILU_TRACE) and summarise the per-CTA timeline."""
import os
import subprocess
import sys

import numpy as np

here = os.path.dirname(os.path.abspath(__file__))
path = "/tmp/tilu_trace.bin"
if os.environ.get("TILU_TRACE") is None:
    env = dict(os.environ, TILU_TRACE=path)
    subprocess.run([sys.executable, os.path.join(here, "prof_batch.py"), "--sweeps", "2"] + sys.argv[1:], env=env,
                   check=True)
raw = open(path, "rb").read()
G, nl, k = np.frombuffer(raw[:12], dtype=np.int32)
t = np.frombuffer(raw[12:], dtype=np.uint64).astype(np.float64).reshape(2, G * nl, k)
for name, tt in (("fwd", t[0]), ("bwd", t[1])):
    t0 = tt[:, 0].min()
    start, open_, end = (tt[:, 0] - t0) / 1e3, (tt[:, 1] - t0) / 1e3, (tt[:, 2] - t0) / 1e3
    waited = tt[:, 3] / 1965.0  # cycles -> us at 1965 MHz
    print(f"{name}: pass {end.max():.1f} us; CTA life mean {np.mean(end - start):.1f} us; "
          f"initial wait mean {np.mean(open_ - start):.1f} us; in-loop waits mean {np.mean(waited):.1f} us")
    # ticket order = layer-major: layer li of group 0 is ticket li * G
    for li in (0, 1, 2, 5, 10, 20, 40, 60, 80, 100, nl - 1):
        if li >= nl:
            continue
        i = li * G
        c = tt[i] / 1965.0
        print(f"   layer#{li:3d} g0: start {start[i]:8.1f} open {open_[i]:8.1f} end {end[i]:8.1f} "
              f"dur {end[i]-open_[i]:7.1f} | us: dep-wait {c[3]:7.1f} release {c[4]:6.1f} w0-bar {c[5]:7.1f} "
              f"w0-steps {c[6]:7.1f} | windows {int(tt[i][7])}")

tail = np.frombuffer(raw[12:], dtype=np.uint64)[-4:].astype(np.float64)
if tail[1] > 0:
    print(f"layer-1 warp-0 profile: {int(tail[1])} row inits, {tail[0]/max(tail[1],1):.0f} cycles each; "
          f"{int(tail[3])} points, {tail[2]/max(tail[3],1):.0f} cycles per point (incl. init)")

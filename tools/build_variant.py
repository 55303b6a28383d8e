"""Build a measurement variant of libtilu.so with extra -D flags (A/B experiments, instrumentation):
    python tools/build_variant.py prof -DTILU_PLANE_PROF          -> paper_2210_15280_b200/lib/variants/libtilu_prof.so
Use it with TILU_LIB=<path>.  Never the product library."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as G  # noqa: E402

tag, flags = sys.argv[1], sys.argv[2:]
out = os.path.join(G.PKG, "lib", "variants", f"libtilu_{tag}.so")
os.makedirs(os.path.dirname(out), exist_ok=True)
srcs = [os.path.join(G.CSRC, s) for s in G.SOURCES]
cmd = [G._nvcc(), *G.NVCC_FLAGS, *flags, "-shared", "-I", os.path.join(ROOT, "include"), "-I", G.CSRC, *srcs, "-o", out]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.stderr.write(r.stdout[-3000:] + r.stderr[-3000:])
    sys.exit(1)
print(out)

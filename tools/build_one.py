"""A/B variant of ONE translation unit: recompile it with extra -D flags and link it with the product build's
other objects:   python tools/build_one.py <tag> tilu_batch.cu -DTILU_BWD_MINB2=5
-> paper_2210_15280_b200/lib/variants/libtilu_<tag>.so  (use with TILU_LIB=<path>; never the product library)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as G  # noqa: E402

tag, unit, flags = sys.argv[1], sys.argv[2], sys.argv[3:]
G.build_lib()
objdir = os.path.join(G.PKG, "lib", "obj")
vdir = os.path.join(G.PKG, "lib", "variants")
os.makedirs(vdir, exist_ok=True)
obj = os.path.join(vdir, f"{unit}.{tag}.o")
inc = ["-I", os.path.join(ROOT, "include"), "-I", G.CSRC]
r = subprocess.run([G._nvcc(), *G.NVCC_FLAGS, *flags, *inc, "-c", os.path.join(G.CSRC, unit), "-o", obj],
                   capture_output=True, text=True)
open(obj + ".log", "w").write(r.stdout + r.stderr)
if r.returncode:
    sys.stderr.write((r.stdout + r.stderr)[-3000:])
    sys.exit(1)
objs = [obj if s == unit else os.path.join(objdir, s + ".o") for s in G.SOURCES]
out = os.path.join(vdir, f"libtilu_{tag}.so")
subprocess.run([G._nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *objs, "-o", out], check=True)
print(out)

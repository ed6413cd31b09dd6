"""Build an alternative liblor_b200.so for A/B timing (scripts/ab_lib.sh): one translation unit
recompiled with extra -D flags, everything else from build/lor.  usage:
    python scripts/alt_build.py lor_xv_nd.cu alt/lib_b_x.so -DND_FENCE=2"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_12253_b200 import build as b  # noqa: E402

tu, out, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
obj = f"/tmp/alt_{os.path.basename(tu)}.o"
r = subprocess.run([b.NVCC] + b.FLAGS + b.ARCH + defs + ["-c", os.path.join(b.CSRC, tu), "-o", obj],
                   capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr[-2000:])
skip = os.path.basename(tu)[:-3] + ".o"
objs = [os.path.join(b.BUILD, f) for f in os.listdir(b.BUILD) if f.endswith(".o") and f != skip] + [obj]
os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
r = subprocess.run([b.NVCC] + b.ARCH + ["-shared", "-o", out] + objs + ["-ldl"], capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr[-2000:])
print("wrote", out)

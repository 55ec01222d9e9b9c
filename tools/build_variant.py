"""Builds a tuning variant of the library with extra nvcc -D flags:
    python tools/build_variant.py NAME -DDFM_S_FWD=6 ...
-> build/variants/libdifform_NAME.so (load it with DFM_LIB=<path>)."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_01249_b200 import build as B

name, args = sys.argv[1], sys.argv[2:]
# "16:-DX=1" applies to the 16-wide instantiation only (kernels_tma16.cu)
defs = [a for a in args if not a.startswith("16:")]
defs16 = defs + [a[3:] for a in args if a.startswith("16:")]
out = os.path.join(B.ROOT, "build", "variants", name)
os.makedirs(out, exist_ok=True)
B.build(verbose=False)
objs = []
for f in sorted(os.listdir(B.CSRC)):
    if not f.endswith(".cu"):
        continue
    src = os.path.join(B.CSRC, f)
    if f in ("kernels_tma.cu", "kernels_tma16.cu", "kernels_brick.cu"):
        obj = os.path.join(out, f.replace(".cu", ".o"))
        extra = defs16 if f == "kernels_tma16.cu" else defs
        subprocess.run([B.NVCC] + B.ARCH + B.FLAGS + extra + ["-c", src, "-o", obj], check=True)
    else:
        obj = os.path.join(B.OBJ, f.replace(".cu", ".o"))
    objs.append(obj)
lib = os.path.join(B.ROOT, "build", "variants", f"libdifform_{name}.so")
subprocess.run([B.NVCC] + B.ARCH + ["-shared", "-cudart", "static", "-o", lib] + objs +
               ["-Xlinker", "--exclude-libs,ALL", "-lrt", "-ldl", "-lpthread"], check=True)
print(lib)

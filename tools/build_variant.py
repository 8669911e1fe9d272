"""Build an A/B variant of libatom: recompile the given sources with extra -D flags and link with
the normal objects into paper_2403_10504_b200/libatom_<tag>.so (select it with ATOM_LIB=...).

    python tools/build_variant.py <tag> <source.cu> [-DNAME=VALUE ...]
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_10504_b200 import build as b  # noqa: E402

tag, src, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
b.build(verbose=False)
objs = sorted(os.path.join(b.BUILD, f) for f in os.listdir(b.BUILD) if f.endswith(".o") and "__" not in f)
vobj = os.path.join(b.BUILD, f"{os.path.basename(src)}__{tag}.o")
subprocess.run([b.NVCC] + b._flags() + defs + ["-c", os.path.join(b.CSRC, src), "-o", vobj], check=True)
objs = [vobj if os.path.basename(o) == os.path.basename(src) + ".o" else o for o in objs]
out = os.path.join(b.HERE, f"libatom_{tag}.so")
_, libdir = b._nccl_dirs()
subprocess.run([b.NVCC] + b.ARCH + ["-shared", "-o", out] + objs +
               ["-L", libdir, "-l:libnccl.so.2", "-Xlinker", f"-rpath={libdir}", "-lpthread"], check=True)
print(out)

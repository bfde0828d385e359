"""Build a variant of libirdn.so with extra nvcc defines into build_variants/ (A/B experiments).

    python tools/build_variant.py NAME -DIRDN_X=0 [...]   ->  build_variants/NAME.so
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1201_3972_b200 import build as B  # noqa: E402

name, extra = sys.argv[1], sys.argv[2:]
os.makedirs(os.path.join(B.REPO, "build_variants"), exist_ok=True)
target = os.path.join(B.REPO, "build_variants", name + ".so")
cmd = [B.NVCC, *B.NVCC_FLAGS, *extra, "-I", os.path.join(B.REPO, "include"), "-o", target,
       *[os.path.join(B.CSRC, f) for f in B.CUDA_SOURCES]]
res = subprocess.run(cmd, capture_output=True, text=True)
open(target + ".log", "w").write(res.stdout + res.stderr)
if res.returncode:
    sys.exit(res.stdout + res.stderr)
print(target)

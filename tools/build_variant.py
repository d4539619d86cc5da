"""Build the library with extra nvcc flags into ab/<name>.so (A/B runs:
DCOMP_LIB=ab/<name>.so python tools/profile_decode.py ...).

    python tools/build_variant.py NAME [-DFOO=1 ...]
"""
import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2502_15443_b200 import _build  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
obj = os.path.join(ROOT, "ab", "obj_" + name)
os.makedirs(obj, exist_ok=True)
srcs = sorted(glob.glob(os.path.join(_build.CSRC, "*.cu")))


def cc(src):
    o = os.path.join(obj, os.path.basename(src)[:-3] + ".o")
    r = subprocess.run([_build.nvcc(), *_build.ARCH, *_build.NVCC_FLAGS, *flags, "-c", src, "-o", o],
                       capture_output=True, text=True)
    if r.returncode:
        raise SystemExit(r.stderr)
    return o


with ThreadPoolExecutor(8) as ex:
    objs = list(ex.map(cc, srcs))
lib = os.path.join(ROOT, "ab", name + ".so")
subprocess.run([_build.nvcc(), *_build.ARCH, "-shared", "-o", lib, *objs, "-lcuda"], check=True)
print(lib)

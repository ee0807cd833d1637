"""Build libspx variants with extra -D flags for A/B kernel experiments (development).

    python tools/build_variants.py name1:-DFOO=1,-DBAR name2:...
    SPX_LIB_VARIANT=variants/libspx_name1.so python bench.py
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1509_04232_b200 import _build as B  # noqa: E402

OBJ = os.path.join(B.REPO, "build", "variants")
OUT = os.path.join(B.REPO, "variants")  # git-ignored, travels with gpurun


def build(name, defs):
    d = os.path.join(OBJ, name)
    os.makedirs(OUT, exist_ok=True)
    os.makedirs(d, exist_ok=True)

    def one(src):
        obj = os.path.join(d, os.path.basename(src) + ".o")
        subprocess.run([B.NVCC, *B.ARCH, *B.FLAGS, *defs, "-c", src, "-o", obj], check=True)
        return obj

    with ThreadPoolExecutor(8) as ex:
        objs = list(ex.map(one, B.sources()))
    lib = os.path.join(OUT, f"libspx_{name}.so")
    subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", lib, *objs, "-Xcompiler", "-fPIC"], check=True)
    print(lib)


for arg in sys.argv[1:]:
    name, _, flags = arg.partition(":")
    build(name, [f for f in flags.split(",") if f])

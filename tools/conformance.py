"""Run the reference's own pytest suite against this package (conformance check).

    python tools/conformance.py prepare   # here: needs /root/reference
    python tools/conformance.py run       # on the GPU box

`prepare` writes a git-ignored scratch tree `_conformance/` holding the
reference's tests (read from /root/reference, not committed) and a `superpix`
shim that re-exports `paper_1509_04232_b200` under the reference's module
names.  The reference's numpy `kernels/pure.py` (its comparison oracle in
test_kernels / test_imgproc) and its `cli.py` (the front-end, out of scope
here) come from the reference build in `oracle/_ref/` and run on top of this
package.  Tests that assert the reference's own implementation names
("compiled", the "pure" fallback, SUPERPIX_PURE) fail by design and are
listed as such in the report.
"""
import os
import shutil
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(REPO, "_conformance")
REF_TESTS = "/root/reference/pkg/tests"
REF_PKG = os.path.join(REPO, "oracle", "_ref", "superpix")

SHIM = '''"""superpix -> paper_1509_04232_b200 (conformance shim, generated)."""
import importlib
import sys

import paper_1509_04232_b200 as _b
from paper_1509_04232_b200 import *  # noqa: F401,F403
from paper_1509_04232_b200 import __all__  # noqa: F401

__version__ = getattr(_b, "__version__", "0.1.0")
for _m in ("engine", "imgproc", "slic_core", "connectivity", "errors"):
    sys.modules[__name__ + "." + _m] = importlib.import_module("paper_1509_04232_b200." + _m)
'''
KERNELS = '''"""superpix.kernels -> paper_1509_04232_b200.kernels (+ the reference's pure oracle)."""
from paper_1509_04232_b200.kernels import ACTIVE, active, get_impl, has_compiled  # noqa: F401

from . import pure, tables  # noqa: F401  (reference numpy implementation, comparison only)
'''


def prepare():
    if os.path.exists(OUT):
        shutil.rmtree(OUT)
    os.makedirs(os.path.join(OUT, "superpix", "kernels"))
    shutil.copytree(REF_TESTS, os.path.join(OUT, "tests"))
    with open(os.path.join(OUT, "superpix", "__init__.py"), "w") as f:
        f.write(SHIM)
    with open(os.path.join(OUT, "superpix", "kernels", "__init__.py"), "w") as f:
        f.write(KERNELS)
    shutil.copy(os.path.join(REF_PKG, "cli.py"), os.path.join(OUT, "superpix", "cli.py"))
    for m in ("pure.py", "tables.py"):
        shutil.copy(os.path.join(REF_PKG, "kernels", m), os.path.join(OUT, "superpix", "kernels", m))
    print("prepared", OUT)


def run():
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([OUT, REPO]))
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(OUT, "tests"), "-q",
                        "-p", "no:cacheprovider", "-rf", "--timeout", "900"], env=env, cwd=OUT)
    return r.returncode


if __name__ == "__main__":
    if sys.argv[1] == "prepare":
        prepare()
    else:
        sys.exit(run())

"""CPU oracle for the SLIC hot path -- TEST INFRASTRUCTURE ONLY.

This package is the parity checker.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.
The product package ``paper_1509_04232_b200`` never imports, links or calls
anything under ``oracle/``.

Two checkers live here:

* ``spx_oracle.c`` -- a plain-C restatement of the reference kernel set
  (``/root/reference/pkg/src/superpix/kernels/_core.pyx``), built to
  ``oracle/libspx_oracle.so`` by :func:`build`.  This module wraps it with the
  reference's kernel-protocol signatures (numpy arrays, band arguments), so
  it can be called exactly like ``superpix.kernels._core``.
* ``oracle/_ref`` -- the unmodified reference package with its Cython kernels
  compiled by ``oracle/build_ref.sh`` (only when ``/root/reference`` is
  present at build time; the built files travel to the GPU box).

Parity of the C restatement is pinned by ``tests/test_oracle.py`` against the
golden vectors in ``tests/golden`` (generated from the reference's compiled
path by ``tests/golden/make_golden.py``) and against ``oracle/_ref``.
"""

import ctypes
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libspx_oracle.so")
REF_DIR = os.path.join(HERE, "_ref")

NAME = "oracle"

_lib = None


def build(force=False):
    """Compile the C restatement (gcc, -ffp-contract=off like pkg/setup.py:13)."""
    src = os.path.join(HERE, "spx_oracle.c")
    if not force and os.path.exists(LIB_PATH) and os.path.getmtime(LIB_PATH) >= os.path.getmtime(src):
        return LIB_PATH
    cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC",
           "-std=c11", src, "-o", LIB_PATH, "-lm"]
    subprocess.check_call(cmd)
    return LIB_PATH


def build_ref():
    """Build oracle/_ref from /root/reference when it exists (see build_ref.sh)."""
    script = os.path.join(HERE, "build_ref.sh")
    env = dict(os.environ, PYTHON=sys.executable)
    subprocess.check_call(["bash", script], env=env)


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        build()
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    I64 = ctypes.c_int64
    D = ctypes.c_double
    I = ctypes.c_int
    sig = {
        "spxo_tables": (None, [P, P, P]),
        "spxo_cbrt_glibc": (D, [D]),
        "spxo_convert_band": (None, [P, P, I64, I64, I, I64, I64]),
        "spxo_init_centers_range": (None, [P, I64, I64, I64, I64, P, P, I64, I64]),
        "spxo_perturb_range": (None, [P, I64, I64, P, P, I64, I64]),
        "spxo_associate_band": (None, [P, I64, I64, P, P, P, I64, I64, I64, D, I64, I64]),
        "spxo_accumulate_range": (None, [P, P, I64, I64, P, I64, I64, I64, I64, I64, I64]),
        "spxo_accumulate_spill": (I64, [P, P, I64, I64, P, I64, I64, I64]),
        "spxo_reduce_range": (None, [P, I64, P, P, P, P, P, I64, I64]),
        "spxo_weak_band": (None, [P, P, I64, I64, I64, I64]),
        "spxo_strict_fill": (I, [P, P, I64, I64, I64]),
        "spxo_center_shift": (D, [P, P, I64]),
        "spxo_segment": (I, [P, I64, I64, I, I64, I64, I64, D, I, I, I, I64, I64, D,
                             P, P, P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _check(a, dtype, ndim=None, writable=False):
    if not isinstance(a, np.ndarray) or a.dtype != dtype or not a.flags.c_contiguous:
        raise ValueError(f"expected C-contiguous {np.dtype(dtype)} array")
    if ndim is not None and a.ndim != ndim:
        raise ValueError(f"expected {ndim}-D array, got {a.ndim}-D")
    if writable and not a.flags.writeable:
        raise ValueError("output array is read-only")
    return a


# ---- kernel protocol (same signatures as _core.pyx) -------------------------

def tables():
    lut = np.empty(256)
    mat = np.empty(9)
    white = np.empty(3)
    _load().spxo_tables(_p(lut), _p(mat), _p(white))
    return lut, mat.reshape(3, 3), white


def cbrt_glibc(x):
    return _load().spxo_cbrt_glibc(float(x))


def convert_band(rgb, out, space, y0, y1):
    _check(rgb, np.uint8, 3)
    _check(out, np.float32, 3, True)
    _load().spxo_convert_band(_p(rgb), _p(out), rgb.shape[0], rgb.shape[1], int(space), y0, y1)


def init_centers_range(img, s, ns_c, cxy, clab, k0, k1):
    _check(img, np.float32, 3)
    _check(cxy, np.float64, 2, True)
    _check(clab, np.float64, 2, True)
    _load().spxo_init_centers_range(_p(img), img.shape[0], img.shape[1], s, ns_c,
                                    _p(cxy), _p(clab), k0, k1)


def perturb_range(img, cxy, clab, k0, k1):
    _check(img, np.float32, 3)
    _check(cxy, np.float64, 2, True)
    _check(clab, np.float64, 2, True)
    _load().spxo_perturb_range(_p(img), img.shape[0], img.shape[1], _p(cxy), _p(clab), k0, k1)


def associate_band(img, cxy, clab, labels, s, ns_r, ns_c, xy_weight, y0, y1):
    _check(img, np.float32, 3)
    _check(cxy, np.float64, 2)
    _check(clab, np.float64, 2)
    _check(labels, np.int32, 2, True)
    _load().spxo_associate_band(_p(img), img.shape[0], img.shape[1], _p(cxy), _p(clab),
                                _p(labels), s, ns_r, ns_c, float(xy_weight), y0, y1)


def accumulate_range(img, labels, slab, s, ns_c, tile_len, k0, k1):
    _check(img, np.float32, 3)
    _check(labels, np.int32, 2)
    _check(slab, np.float64, 3, True)
    _load().spxo_accumulate_range(_p(img), _p(labels), labels.shape[0], labels.shape[1],
                                  _p(slab), slab.shape[1], s, ns_c, tile_len, k0, k1)


def accumulate_spill(img, labels, slab, s, ns_c):
    _check(img, np.float32, 3)
    _check(labels, np.int32, 2)
    _check(slab, np.float64, 3, True)
    return int(_load().spxo_accumulate_spill(_p(img), _p(labels), labels.shape[0],
                                             labels.shape[1], _p(slab), slab.shape[1], s, ns_c))


def reduce_range(slab, prev_xy, prev_lab, out_xy, out_lab, out_counts, k0, k1):
    _check(slab, np.float64, 3, True)
    _load().spxo_reduce_range(_p(slab), slab.shape[1], _p(_check(prev_xy, np.float64)),
                              _p(_check(prev_lab, np.float64)),
                              _p(_check(out_xy, np.float64, writable=True)),
                              _p(_check(out_lab, np.float64, writable=True)),
                              _p(_check(out_counts, np.int64, writable=True)), k0, k1)


def weak_band(src, dst, y0, y1):
    _check(src, np.int32, 2)
    _check(dst, np.int32, 2, True)
    _load().spxo_weak_band(_p(src), _p(dst), src.shape[0], src.shape[1], y0, y1)


def strict_fill(src, dst, min_size):
    _check(src, np.int32, 2)
    _check(dst, np.int32, 2, True)
    if _load().spxo_strict_fill(_p(src), _p(dst), src.shape[0], src.shape[1], min_size) != 0:
        raise MemoryError()


def center_shift(new_xy, old_xy):
    new_xy = np.ascontiguousarray(new_xy, dtype=np.float64)
    old_xy = np.ascontiguousarray(old_xy, dtype=np.float64)
    return _load().spxo_center_shift(_p(new_xy), _p(old_xy), new_xy.shape[0])


def segment(rgb, s, ns_r, ns_c, compactness, no_iters=5, space=2, perturb=False,
            connectivity=1, min_size=None, tile_len=16, early_stop=None):
    """Whole-frame pipeline (engine.py:125-230).  Returns (labels, cxy, clab, counts, passes)."""
    _check(rgb, np.uint8, 3)
    h, w = rgb.shape[0], rgb.shape[1]
    k = ns_r * ns_c
    labels = np.empty((h, w), dtype=np.int32)
    cxy = np.empty((k, 2))
    clab = np.empty((k, 3))
    counts = np.empty(k, dtype=np.int64)
    if min_size is None:
        min_size = max(1, s * s // 4)
    rc = _load().spxo_segment(_p(rgb), h, w, space, s, ns_r, ns_c, compactness / s, no_iters,
                              int(perturb), connectivity, min_size, tile_len,
                              -1.0 if early_stop is None else float(early_stop),
                              _p(labels), _p(cxy), _p(clab), _p(counts))
    if rc < 0:
        raise MemoryError()
    return labels, cxy, clab, counts, rc


def reference_package():
    """Import the built reference package from oracle/_ref (None if absent)."""
    if not os.path.isdir(os.path.join(REF_DIR, "superpix")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import superpix  # noqa: E402
    return superpix

"""CUDA kernel set with the reference kernel-plugin protocol.

Same nine functions, signatures and in-place band semantics as
superpix/kernels/_core.pyx (listed in SURVEY.md §8(b)); each forwards to the
matching ``spx_*`` entry point of libspx.so (include/spx.h).

Arguments may be numpy arrays (the reference's calling convention: the
array is staged to the GPU, the kernel runs, and only the band/range the
call owns is copied back) or CUDA ``torch.Tensor``s (zero-copy, enqueued on
the current torch stream).  Dtype/contiguity mismatches raise ValueError,
as Cython's typed memoryviews do.
"""

import ctypes

import numpy as np

from .. import _lib

NAME = "cuda"

_TORCH_DTYPES = None


def _torch():
    import torch
    return torch


def _np_to_torch_dtype(dt):
    torch = _torch()
    return {np.dtype(np.uint8): torch.uint8, np.dtype(np.float32): torch.float32,
            np.dtype(np.float64): torch.float64, np.dtype(np.int32): torch.int32,
            np.dtype(np.int64): torch.int64}[np.dtype(dt)]


class _Arg:
    """A kernel argument resident on the GPU (staged from numpy if needed)."""

    __slots__ = ("host", "dev")

    def __init__(self, a, dtype, ndim, name, writable=False):
        torch = _torch()
        if isinstance(a, torch.Tensor):
            if not a.is_cuda:
                raise ValueError(f"{name}: torch tensors must live on a CUDA device")
            if a.dtype != _np_to_torch_dtype(dtype):
                raise ValueError(f"{name}: buffer dtype mismatch, expected {np.dtype(dtype)}")
            if ndim is not None and a.dim() != ndim:
                raise ValueError(f"{name}: buffer has wrong number of dimensions "
                                 f"(expected {ndim}, got {a.dim()})")
            if not a.is_contiguous():
                raise ValueError(f"{name}: ndarray is not C-contiguous")
            self.host = None
            self.dev = a
            return
        if not isinstance(a, np.ndarray):
            raise ValueError(f"{name}: expected a numpy array or CUDA tensor")
        if a.dtype != np.dtype(dtype):
            raise ValueError(f"{name}: buffer dtype mismatch, expected {np.dtype(dtype)} "
                             f"but got {a.dtype}")
        if ndim is not None and a.ndim != ndim:
            raise ValueError(f"{name}: buffer has wrong number of dimensions "
                             f"(expected {ndim}, got {a.ndim})")
        if not a.flags.c_contiguous:
            raise ValueError(f"{name}: ndarray is not C-contiguous")
        if writable and not a.flags.writeable:
            raise ValueError(f"{name}: buffer source array is read-only")
        self.host = a
        src = a if a.flags.writeable else a.copy()
        self.dev = torch.from_numpy(src).to("cuda", non_blocking=False) if a.size else \
            torch.empty(a.shape, dtype=_np_to_torch_dtype(dtype), device="cuda")

    @property
    def ptr(self):
        return ctypes.c_void_p(self.dev.data_ptr())

    def copy_back(self, sl=slice(None)):
        """Copy dev[sl] (along the first axis) back into the numpy array."""
        if self.host is None:
            return
        part = self.dev[sl]
        if part.numel():
            self.host[sl] = part.cpu().numpy()

    @property
    def shape(self):
        return tuple(self.dev.shape)


def _stream():
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _call(fn, *args, what=""):
    lib = _lib.load()
    _lib.check(getattr(lib, fn)(*args), what or fn)


# ---- the protocol --------------------------------------------------------------

def convert_band(rgb, out, space, y0, y1):
    """_core.pyx:45-83: rows [y0, y1) of an 8-bit RGB raster into `out`."""
    r = _Arg(rgb, np.uint8, 3, "rgb")
    o = _Arg(out, np.float32, 3, "out", writable=True)
    h, w = r.shape[0], r.shape[1]
    if o.shape != (h, w, 3) or r.shape[2] != 3:
        raise ValueError("convert_band: rgb and out must both be (h, w, 3)")
    _call("spx_convert_band", r.ptr, o.ptr, h, w, int(space), int(y0), int(y1), _stream())
    o.copy_back(slice(y0, y1))


def init_centers_range(img, s, ns_c, cxy, clab, k0, k1):
    """_core.pyx:86-107: seed centres [k0, k1) at (clamped) cell centres."""
    im = _Arg(img, np.float32, 3, "img")
    xy = _Arg(cxy, np.float64, 2, "cxy", writable=True)
    lab = _Arg(clab, np.float64, 2, "clab", writable=True)
    _check_rows(xy, lab, k1)
    _call("spx_init_centers_range", im.ptr, im.shape[0], im.shape[1], int(s), int(ns_c), xy.ptr,
          lab.ptr, int(k0), int(k1), _stream())
    xy.copy_back(slice(k0, k1))
    lab.copy_back(slice(k0, k1))


def perturb_range(img, cxy, clab, k0, k1):
    """_core.pyx:123-156: move centres [k0, k1) to their 3x3 gradient minimum."""
    im = _Arg(img, np.float32, 3, "img")
    xy = _Arg(cxy, np.float64, 2, "cxy", writable=True)
    lab = _Arg(clab, np.float64, 2, "clab", writable=True)
    _check_rows(xy, lab, k1)
    _call("spx_perturb_range", im.ptr, im.shape[0], im.shape[1], xy.ptr, lab.ptr, int(k0),
          int(k1), _stream())
    xy.copy_back(slice(k0, k1))
    lab.copy_back(slice(k0, k1))


def associate_band(img, cxy, clab, labels, s, ns_r, ns_c, xy_weight, y0, y1):
    """_core.pyx:172-197: label rows [y0, y1) with the best of <= 9 centres."""
    im = _Arg(img, np.float32, 3, "img")
    xy = _Arg(cxy, np.float64, 2, "cxy")
    lab = _Arg(clab, np.float64, 2, "clab")
    lb = _Arg(labels, np.int32, 2, "labels", writable=True)
    n = min(xy.shape[0], lab.shape[0])
    _call("spx_associate_band", im.ptr, im.shape[0], lb.shape[1], xy.ptr, lab.ptr, n, lb.ptr,
          int(s), int(ns_r), int(ns_c), float(xy_weight), int(y0), int(y1), _stream())
    lb.copy_back(slice(y0, y1))


def accumulate_range(img, labels, slab, s, ns_c, tile_len, k0, k1):
    """_core.pyx:200-255: per-strip partial sums of clusters [k0, k1)."""
    im = _Arg(img, np.float32, 3, "img")
    lb = _Arg(labels, np.int32, 2, "labels")
    sb = _Arg(slab, np.float64, 3, "slab", writable=True)
    if k1 > sb.shape[0]:
        raise ValueError("accumulate_range: cluster range exceeds slab rows")
    _call("spx_accumulate_range", im.ptr, lb.ptr, lb.shape[0], lb.shape[1], sb.ptr, sb.shape[1],
          int(s), int(ns_c), int(tile_len), int(k0), int(k1), _stream())
    sb.copy_back(slice(k0, k1))


def accumulate_spill(img, labels, slab, s, ns_c):
    """_core.pyx:258-285: add out-of-window pixels to strip 0; returns the count."""
    im = _Arg(img, np.float32, 3, "img")
    lb = _Arg(labels, np.int32, 2, "labels")
    sb = _Arg(slab, np.float64, 3, "slab", writable=True)
    spills = ctypes.c_int64(0)
    _call("spx_accumulate_spill", im.ptr, lb.ptr, lb.shape[0], lb.shape[1], sb.ptr, sb.shape[0],
          sb.shape[1], int(s), int(ns_c), ctypes.byref(spills), _stream())
    if spills.value:
        sb.copy_back()
    return int(spills.value)


def reduce_range(slab, prev_xy, prev_lab, out_xy, out_lab, out_counts, k0, k1):
    """_core.pyx:288-325: pairwise-tree reduce of clusters [k0, k1) (destroys slab rows)."""
    sb = _Arg(slab, np.float64, 3, "slab", writable=True)
    pxy = _Arg(prev_xy, np.float64, 2, "prev_xy")
    plab = _Arg(prev_lab, np.float64, 2, "prev_lab")
    oxy = _Arg(out_xy, np.float64, 2, "out_xy", writable=True)
    olab = _Arg(out_lab, np.float64, 2, "out_lab", writable=True)
    ocnt = _Arg(out_counts, np.int64, 1, "out_counts", writable=True)
    for a in (pxy, plab, oxy, olab, ocnt):
        if k1 > a.shape[0]:
            raise ValueError("reduce_range: cluster range exceeds array rows")
    _call("spx_reduce_range", sb.ptr, sb.shape[1], pxy.ptr, plab.ptr, oxy.ptr, olab.ptr, ocnt.ptr,
          int(k0), int(k1), _stream())
    for a in (sb, oxy, olab, ocnt):
        a.copy_back(slice(k0, k1))


def weak_band(src, dst, y0, y1):
    """_core.pyx:328-356: one stray-pixel pass over rows [y0, y1)."""
    s = _Arg(src, np.int32, 2, "src")
    d = _Arg(dst, np.int32, 2, "dst", writable=True)
    if s.shape != d.shape:
        raise ValueError("weak_band: src and dst shapes differ")
    _call("spx_weak_band", s.ptr, d.ptr, s.shape[0], s.shape[1], int(y0), int(y1), _stream())
    d.copy_back(slice(y0, y1))


def strict_fill(src, dst, min_size):
    """_core.pyx:359-461: scan-order component fill (parallel, same result)."""
    s = _Arg(src, np.int32, 2, "src")
    d = _Arg(dst, np.int32, 2, "dst", writable=True)
    if s.shape != d.shape:
        raise ValueError("strict_fill: src and dst shapes differ")
    _call("spx_strict_fill", s.ptr, d.ptr, s.shape[0], s.shape[1], int(min_size), _stream())
    d.copy_back()


def _check_rows(xy, lab, k1):
    if k1 > xy.shape[0] or k1 > lab.shape[0]:
        raise ValueError("cluster range exceeds centre array rows")

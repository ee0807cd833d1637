"""Kernel-plugin selector (mirrors superpix/kernels/__init__.py:12-44).

There is exactly one implementation, the CUDA kernel set in libspx.so.  The
reference's names keep working: "auto" and "compiled" select it; "cuda" is
its own name.  "pure" (the reference's numpy fallback) does not exist here --
asking for it raises ImportError, the same error the reference raises for a
missing implementation.  Unknown names raise ValueError.
"""

from . import cuda

ACTIVE = cuda


def active():
    """Name of the selected implementation: "cuda"."""
    return ACTIVE.NAME


def has_compiled():
    """True when the native library loads (it is required, not optional)."""
    try:
        from .. import _lib
        _lib.load()
        return True
    except ImportError:
        return False


def get_impl(which="auto"):
    """Return a kernel module by name ("auto", "cuda" or "compiled")."""
    if which in ("auto", "cuda", "compiled"):
        return cuda
    if which == "pure":
        raise ImportError("this package has no CPU kernel implementation; use 'cuda'")
    raise ValueError(f"unknown kernel implementation {which!r}")

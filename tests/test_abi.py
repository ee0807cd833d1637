"""The C ABI library loads and exports exactly what include/spx.h declares.

CPU-only: no compute calls are made (there is no GPU here); the only calls
are host-side queries.  Also pins the host colour tables the kernels use to
the oracle / reference tables.py values.
"""

import ctypes
import os
import re

import numpy as np
import pytest

import oracle
from paper_1509_04232_b200 import _lib

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "spx.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"SPX_API\s+[\w\s\*]+?\b(spx_\w+)\s*\(", text)))


def test_library_exists_and_loads():
    assert os.path.exists(_lib.LIB_PATH), "build libspx.so first (__graft_entry__.build())"
    lib = _lib.load()
    assert lib.spx_name() == b"cuda"
    assert lib.spx_abi_version() == 1


def test_every_declared_symbol_is_exported_and_bound():
    syms = declared_symbols()
    assert len(syms) >= 20
    raw = ctypes.CDLL(_lib.LIB_PATH)
    for s in syms:
        assert hasattr(raw, s), f"{s} declared in spx.h but not exported"
        assert s in _lib.SIGNATURES, f"{s} has no ctypes signature"
    assert set(_lib.SIGNATURES) == set(syms)


def test_exports_are_only_the_abi():
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert {s for s in exported if s.startswith("spx_")} == set(declared_symbols())


def test_host_tables_match_reference_tables():
    lut = np.empty(256); mat = np.empty(9); white = np.empty(3)
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    _lib.check(_lib.load().spx_debug_tables(p(lut), p(mat), p(white)))
    olut, omat, owhite = oracle.tables()
    assert lut.tobytes() == olut.tobytes()
    assert mat.tobytes() == omat.ravel().tobytes()
    assert white.tobytes() == owhite.tobytes()
    sp = oracle.reference_package()
    if sp is not None:
        from superpix.kernels import tables
        assert lut.tobytes() == tables.LINEAR_LUT.tobytes()
        assert white.tobytes() == tables.WHITE.tobytes()


def test_status_codes_map_to_reference_exceptions():
    from paper_1509_04232_b200.errors import DimensionMismatchError, InvalidSettingsError
    with pytest.raises(InvalidSettingsError):
        _lib.check(_lib.SPX_ERR_INVALID_SETTINGS)
    with pytest.raises(DimensionMismatchError):
        _lib.check(_lib.SPX_ERR_DIMENSION)
    with pytest.raises(MemoryError):
        _lib.check(_lib.SPX_ERR_NOMEM)
    with pytest.raises(ValueError):
        _lib.check(_lib.SPX_ERR_VALUE)
    with pytest.raises(_lib.SpxCudaError):
        _lib.check(_lib.SPX_ERR_CUDA)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_1509_04232_b200 as spx
    st = spx.Settings(img_width=8, img_height=8, num_superpixels=4)
    with pytest.raises(_lib.SpxCudaError):
        spx.SegEngine(st)
    with pytest.raises(Exception):
        spx.convert_color_space(spx.ImageRGB(np.zeros((2, 2, 3), np.uint8)), spx.ColorSpace.LAB)


def test_product_never_imports_oracle():
    pkg = os.path.join(REPO, "paper_1509_04232_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(root, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "spx_oracle" not in text, f

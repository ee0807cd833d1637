"""Per-kernel parity: CUDA kernel protocol vs the CPU oracle (bit-exact).

Mirrors the reference's cross-implementation suite (pkg/tests/test_kernels.py):
same seeded inputs, shuffled band splits, plus golden vectors produced by
the reference itself and larger randomized cases.  Runs on a B200 (-m gpu).
"""

import ctypes

import numpy as np
import pytest

import oracle
from paper_1509_04232_b200 import _lib, kernels
from paper_1509_04232_b200.kernels import cuda as K

pytestmark = pytest.mark.gpu


def bits_equal(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and a.tobytes() == b.tobytes()


def split(fn, bounds, *args):
    for lo, hi in bounds:
        fn(*args, lo, hi)


def rand_img(rng, h, w):
    return np.ascontiguousarray(rng.random((h, w, 3), dtype=np.float32) * 100.0)


def make_centers(rng, k, w, h):
    cxy = np.column_stack([rng.random(k) * w, rng.random(k) * h])
    return np.ascontiguousarray(cxy), rng.random((k, 3)) * 100.0


def test_selected_and_named():
    assert kernels.active() == "cuda"
    assert kernels.get_impl("compiled") is K
    assert _lib.load().spx_name() == b"cuda"


def test_filter_sqrt_error_within_bound():
    v = ctypes.c_double()
    _lib.check(_lib.load().spx_debug_sqrt_error(ctypes.byref(v)))
    assert 0 < v.value <= 2.0 ** -21, v.value


def test_update_division_fast_path_is_ieee():
    """The centre update's branch-free division (the compiler's own fast path,
    unrolled) equals IEEE division whenever its guard accepts the operands."""
    out = (ctypes.c_int64 * 2)()
    _lib.check(_lib.load().spx_debug_ddiv_check(1 << 28, 12345, out))
    assert out[0] == 0, f"{out[0]} of {out[1]} fast-path quotients differ"
    assert out[1] > (1 << 26)


@pytest.mark.parametrize("space", [0, 1, 2])
def test_convert_golden_and_bands(golden, space):
    rgb = golden["convert_rgb"]
    out = np.empty(rgb.shape, np.float32)
    split(K.convert_band, [(9, 17), (0, 4), (4, 9)], rgb, out, space)
    assert bits_equal(out, golden[f"convert_out_{space}"])


@pytest.mark.parametrize("space", [0, 1, 2])
def test_convert_all_colours_bitexact(space):
    import torch
    c = np.arange(1 << 24, dtype=np.uint32)
    rgb = np.stack([(c >> 16) & 255, (c >> 8) & 255, c & 255], -1).astype(np.uint8)
    rgb = rgb.reshape(4096, 4096, 3)
    want = np.empty((4096, 4096, 3), np.float32)
    oracle.convert_band(rgb, want, space, 0, 4096)
    d_rgb = torch.from_numpy(rgb).cuda()
    d_out = torch.empty((4096, 4096, 3), dtype=torch.float32, device="cuda")
    K.convert_band(d_rgb, d_out, space, 0, 4096)
    got = d_out.cpu().numpy()
    bad = int((got.view(np.uint32) != want.view(np.uint32)).any(axis=2).sum())
    assert bad == 0, f"{bad} of 2^24 colours differ"


def test_convert_unaligned_band():
    rng = np.random.default_rng(3)
    rgb = rng.integers(0, 256, (37, 41, 3), dtype=np.uint8)
    want = np.empty((37, 41, 3), np.float32)
    oracle.convert_band(rgb, want, 2, 0, 37)
    got = np.empty_like(want)
    split(K.convert_band, [(0, 5), (5, 6), (6, 37)], rgb, got, 2)
    assert bits_equal(got, want)


def test_init_perturb_golden(golden):
    cxy = np.zeros((20, 2)); clab = np.zeros((20, 3))
    split(K.init_centers_range, [(14, 20), (0, 14)], golden["init_img"], 7, 5, cxy, clab)
    assert bits_equal(cxy, golden["init_cxy"]) and bits_equal(clab, golden["init_clab"])
    cxy = golden["perturb_in_xy"].copy(); clab = golden["perturb_in_lab"].copy()
    split(K.perturb_range, [(0, 3), (3, 20)], golden["perturb_img"], cxy, clab)
    assert bits_equal(cxy, golden["perturb_xy"]) and bits_equal(clab, golden["perturb_lab"])


def test_associate_golden(golden):
    img = golden["assoc_img"]
    lab = np.empty(img.shape[:2], np.int32)
    split(K.associate_band, [(11, 29), (0, 11)], img, golden["assoc_cxy"], golden["assoc_clab"],
          lab, 6, 5, 6, 1.7)
    assert bits_equal(lab, golden["assoc_labels"])


@pytest.mark.parametrize("seed", range(6))
def test_associate_random_vs_oracle(seed):
    rng = np.random.default_rng(100 + seed)
    h, w = int(rng.integers(20, 300)), int(rng.integers(20, 300))
    s = int(rng.integers(2, 40))
    ns_r, ns_c = -(-h // s), -(-w // s)
    img = rand_img(rng, h, w)
    cxy, clab = make_centers(rng, ns_r * ns_c, w, h)
    xw = float(rng.choice([0.05, 0.7, 1.7, 10.0]))
    want = np.empty((h, w), np.int32); got = np.empty((h, w), np.int32)
    oracle.associate_band(img, cxy, clab, want, s, ns_r, ns_c, xw, 0, h)
    K.associate_band(img, cxy, clab, got, s, ns_r, ns_c, xw, 0, h)
    assert bits_equal(got, want)


def test_associate_exact_ties_and_flat():
    # flat image + seeded centres: every pixel ties on colour; the tie test of
    # test_slic_core.py:231-246 (pixel (32, 8) -> label 3).
    img = np.zeros((16, 40, 3), np.float32)
    cxy = np.zeros((10, 2)); clab = np.zeros((10, 3))
    oracle.init_centers_range(img, 8, 5, cxy, clab, 0, 10)
    cxy[8] = (28.0, 15.0)
    for far in (2, 7, 9):
        cxy[far] = (1000.0, 1000.0)
    got = np.empty((16, 40), np.int32); want = np.empty_like(got)
    K.associate_band(img, cxy, clab, got, 8, 2, 5, 10.0 / 8, 0, 16)
    oracle.associate_band(img, cxy, clab, want, 8, 2, 5, 10.0 / 8, 0, 16)
    assert bits_equal(got, want) and got[8, 32] == 3


def test_associate_nonfinite_inputs_follow_reference():
    rng = np.random.default_rng(9)
    h, w, s = 24, 24, 6
    img = rand_img(rng, h, w)
    img[3, 4, 0] = np.nan
    img[10, 10, 1] = np.inf
    cxy, clab = make_centers(rng, 16, w, h)
    clab[5, 2] = np.nan
    cxy[9, 0] = np.inf
    got = np.empty((h, w), np.int32); want = np.empty_like(got)
    K.associate_band(img, cxy, clab, got, s, 4, 4, 0.9, 0, h)
    oracle.associate_band(img, cxy, clab, want, s, 4, 4, 0.9, 0, h)
    assert bits_equal(got, want)


def test_associate_large_coordinates():
    # centres far from the origin exercise the tile-relative fp32 coordinates
    rng = np.random.default_rng(11)
    h, w, s = 64, 4000, 16
    img = rand_img(rng, h, w)
    ns_r, ns_c = 4, 250
    cxy, clab = make_centers(rng, ns_r * ns_c, w, h)
    got = np.empty((h, w), np.int32); want = np.empty_like(got)
    K.associate_band(img, cxy, clab, got, s, ns_r, ns_c, 0.625, 0, h)
    oracle.associate_band(img, cxy, clab, want, s, ns_r, ns_c, 0.625, 0, h)
    assert bits_equal(got, want)


def test_accumulate_spill_golden(golden):
    img, labels = golden["accum_img"], golden["accum_labels"]
    slab = np.zeros(golden["accum_slab"].shape)
    split(K.accumulate_range, [(7, 20), (0, 7)], img, labels, slab, 5, 4, 4)
    assert bits_equal(slab, golden["accum_range_slab"])
    spills = K.accumulate_spill(img, labels, slab, 5, 4)
    assert spills == int(golden["accum_spills"])
    assert bits_equal(slab, golden["accum_slab"])


@pytest.mark.parametrize("seed", range(4))
def test_accumulate_random_vs_oracle(seed):
    rng = np.random.default_rng(200 + seed)
    h, w = int(rng.integers(10, 120)), int(rng.integers(10, 120))
    s = int(rng.integers(2, 12))
    tile = int(rng.integers(1, 20))
    ns_r, ns_c = -(-h // s), -(-w // s)
    k = ns_r * ns_c
    img = rand_img(rng, h, w)
    labels = rng.integers(0, k, (h, w)).astype(np.int32)
    n_bl = -(-3 * s // tile)
    a = np.zeros((k, n_bl, 6)); b = np.zeros((k, n_bl, 6))
    oracle.accumulate_range(img, labels, a, s, ns_c, tile, 0, k)
    sa = oracle.accumulate_spill(img, labels, a, s, ns_c)
    K.accumulate_range(img, labels, b, s, ns_c, tile, 0, k)
    sb = K.accumulate_spill(img, labels, b, s, ns_c)
    assert sa == sb
    assert bits_equal(a, b)


@pytest.mark.parametrize("n_bl", [1, 2, 3, 5, 6, 8])
def test_reduce_golden(golden, n_bl):
    g = lambda s: golden[f"reduce{n_bl}_{s}"]  # noqa: E731
    work = g("slab").copy()
    k = work.shape[0]
    oxy = np.zeros((k, 2)); olab = np.zeros((k, 3)); ocnt = np.zeros(k, np.int64)
    split(K.reduce_range, [(4, 7), (0, 4)], work, g("prev_xy"), g("prev_lab"), oxy, olab, ocnt)
    assert bits_equal(oxy, g("xy")) and bits_equal(olab, g("lab")) and bits_equal(ocnt, g("cnt"))


def test_weak_golden_and_random(golden):
    src = golden["weak_src"]
    dst = np.empty_like(src)
    split(K.weak_band, [(0, 6), (13, 19), (6, 13)], src, dst)
    assert bits_equal(dst, golden["weak_dst"])
    rng = np.random.default_rng(5)
    for h, w in ((1, 1), (1, 7), (9, 1), (33, 65), (200, 130)):
        src = rng.integers(0, 3, (h, w)).astype(np.int32)
        a = np.empty_like(src); b = np.empty_like(src)
        oracle.weak_band(src, a, 0, h)
        K.weak_band(src, b, 0, h)
        assert bits_equal(a, b), (h, w)


def test_strict_golden_and_random(golden):
    for name, ms in (("strict", 4), ("strict2", 7)):
        src = golden[f"{name}_src"]
        dst = np.empty_like(src)
        K.strict_fill(src, dst, ms)
        assert bits_equal(dst, golden[f"{name}_dst"]), name
    rng = np.random.default_rng(6)
    for h, w, nl, ms in ((1, 1, 1, 1), (1, 9, 3, 2), (17, 13, 5, 4), (64, 80, 30, 7),
                         (120, 160, 4, 20), (200, 300, 1000, 3)):
        src = rng.integers(0, nl, (h, w)).astype(np.int32)
        a = np.empty_like(src); b = np.empty_like(src)
        oracle.strict_fill(src, a, ms)
        K.strict_fill(src, b, ms)
        assert bits_equal(a, b), (h, w, nl, ms)


def test_torch_tensors_zero_copy():
    import torch
    rng = np.random.default_rng(8)
    rgb = rng.integers(0, 256, (48, 64, 3), dtype=np.uint8)
    want = np.empty((48, 64, 3), np.float32)
    oracle.convert_band(rgb, want, 2, 0, 48)
    d = torch.from_numpy(rgb).cuda()
    out = torch.empty((48, 64, 3), dtype=torch.float32, device="cuda")
    K.convert_band(d, out, 2, 0, 48)
    assert bits_equal(out.cpu().numpy(), want)


def test_dtype_mismatch_raises_valueerror():
    with pytest.raises(ValueError):
        K.convert_band(np.zeros((4, 4, 3), np.int16), np.zeros((4, 4, 3), np.float32), 2, 0, 4)
    with pytest.raises(ValueError):
        K.weak_band(np.zeros((4, 4), np.int64), np.zeros((4, 4), np.int32), 0, 4)

"""Pin the CPU oracle (oracle/spx_oracle.c) to the reference.

CPU-only.  Checks the C restatement against the golden vectors generated from
the reference's compiled path (tests/golden/make_golden.py), and -- when the
reference is built in oracle/_ref -- directly against the reference kernels
on fresh random inputs.
"""

import ctypes
import hashlib

import numpy as np
import pytest

import oracle
from oracle import _check  # noqa: F401


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def bits_equal(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and a.tobytes() == b.tobytes()


@pytest.fixture(scope="module", autouse=True)
def _built():
    oracle.build()


def test_tables_match_reference_expressions():
    lut, mat, white = oracle.tables()
    # tables.py:42-51 in plain Python (same libm pow as the reference)
    expect = []
    for v in range(256):
        c = v / 255.0
        expect.append(c / 12.92 if c <= 0.04045 else ((c + 0.055) / 1.055) ** 2.4)
    assert bits_equal(lut, np.array(expect))
    assert white[1] == (mat[1, 0] + mat[1, 1]) + mat[1, 2]


def test_cbrt_restatement_matches_libm():
    libm = ctypes.CDLL("libm.so.6")
    libm.cbrt.restype = ctypes.c_double
    libm.cbrt.argtypes = [ctypes.c_double]
    rng = np.random.default_rng(7)
    xs = np.concatenate([rng.random(20000) * 1.2, 10.0 ** rng.uniform(-300, 300, 2000),
                         -rng.random(200), [0.0, -0.0, 1.0, 8.0, 0.008856451679035631]])
    bad = [x for x in xs if oracle.cbrt_glibc(float(x)) != libm.cbrt(float(x))]
    assert not bad


@pytest.mark.parametrize("space", [0, 1, 2])
def test_convert_golden(golden, space):
    rgb = golden["convert_rgb"]
    out = np.empty(rgb.shape, np.float32)
    oracle.convert_band(rgb, out, space, 0, rgb.shape[0])
    assert bits_equal(out, golden[f"convert_out_{space}"])


def test_convert_named_colours(golden):
    rgb = golden["convert_named_rgb"]
    out = np.empty(rgb.shape, np.float32)
    oracle.convert_band(rgb, out, 2, 0, 1)
    assert bits_equal(out, golden["convert_named_lab"])
    # test_imgproc.py:19 golden triple, +-1e-3
    assert np.abs(out[0, 0] - np.array([34.7248138153, 25.0000395690, 31.3720602260])).max() < 1e-3


@pytest.mark.parametrize("space", [0, 1, 2])
def test_convert_all_colours_hash(golden_meta, space):
    c = np.arange(1 << 24, dtype=np.uint32)
    rgb = np.stack([(c >> 16) & 255, (c >> 8) & 255, c & 255], -1).astype(np.uint8)
    rgb = rgb.reshape(4096, 4096, 3)
    out = np.empty((4096, 4096, 3), np.float32)
    oracle.convert_band(rgb, out, space, 0, 4096)
    assert sha(out) == golden_meta["hashes"][f"convert_all_colours_space{space}"]


def test_init_and_perturb_golden(golden):
    img = golden["init_img"]
    cxy = np.zeros((20, 2)); clab = np.zeros((20, 3))
    oracle.init_centers_range(img, 7, 5, cxy, clab, 0, 20)
    assert bits_equal(cxy, golden["init_cxy"]) and bits_equal(clab, golden["init_clab"])
    img = golden["perturb_img"]
    cxy = golden["perturb_in_xy"].copy(); clab = golden["perturb_in_lab"].copy()
    oracle.perturb_range(img, cxy, clab, 0, 20)
    assert bits_equal(cxy, golden["perturb_xy"]) and bits_equal(clab, golden["perturb_lab"])


def test_associate_golden(golden):
    img = golden["assoc_img"]
    lab = np.empty(img.shape[:2], np.int32)
    # split bands out of order like test_kernels.py:104
    for y0, y1 in ((11, 29), (0, 11)):
        oracle.associate_band(img, golden["assoc_cxy"], golden["assoc_clab"], lab, 6, 5, 6, 1.7, y0, y1)
    assert bits_equal(lab, golden["assoc_labels"])


def test_accumulate_and_spill_golden(golden):
    img, labels = golden["accum_img"], golden["accum_labels"]
    slab = np.zeros(golden["accum_slab"].shape)
    for k0, k1 in ((7, 20), (0, 7)):
        oracle.accumulate_range(img, labels, slab, 5, 4, 4, k0, k1)
    assert bits_equal(slab, golden["accum_range_slab"])
    spills = oracle.accumulate_spill(img, labels, slab, 5, 4)
    assert spills == int(golden["accum_spills"]) and spills > 0
    assert bits_equal(slab, golden["accum_slab"])


@pytest.mark.parametrize("n_bl", [1, 2, 3, 5, 6, 8])
def test_reduce_golden(golden, n_bl):
    g = lambda s: golden[f"reduce{n_bl}_{s}"]  # noqa: E731
    work = g("slab").copy()
    k = work.shape[0]
    oxy = np.zeros((k, 2)); olab = np.zeros((k, 3)); ocnt = np.zeros(k, np.int64)
    oracle.reduce_range(work, g("prev_xy"), g("prev_lab"), oxy, olab, ocnt, 0, k)
    assert bits_equal(oxy, g("xy")) and bits_equal(olab, g("lab")) and bits_equal(ocnt, g("cnt"))


def test_weak_and_strict_golden(golden):
    src = golden["weak_src"]
    dst = np.empty_like(src)
    for y0, y1 in ((0, 6), (13, 19), (6, 13)):
        oracle.weak_band(src, dst, y0, y1)
    assert bits_equal(dst, golden["weak_dst"])
    for name, ms in (("strict", 4), ("strict2", 7)):
        src = golden[f"{name}_src"]
        dst = np.empty_like(src)
        oracle.strict_fill(src, dst, ms)
        assert bits_equal(dst, golden[f"{name}_dst"])


def _grid(w, h, kw):
    import math
    if "spixel_size" in kw:
        s = kw["spixel_size"]
    else:
        s = max(1, math.floor(math.sqrt(w * h / kw["num_superpixels"]) + 0.5))
    return s, -(-h // s), -(-w // s)


def test_pipeline_golden(golden, golden_meta):
    conn_code = {"weak": 1, "strict": 2}
    space_code = {"rgb": 0, "xyz": 1, "lab": 2}
    for name, w, h, kw, _seed in golden_meta["pipeline_cases"]:
        s, ns_r, ns_c = _grid(w, h, kw)
        conn = 0 if kw.get("do_enforce_connectivity") is False else conn_code[kw.get("connectivity_mode", "weak")]
        labels, cxy, clab, counts, passes = oracle.segment(
            golden[f"pipe_{name}_rgb"], s, ns_r, ns_c, kw.get("compactness", 10.0),
            no_iters=kw.get("no_iters", 5), space=space_code[kw.get("color_space", "lab")],
            perturb=kw.get("enable_perturbation", False), connectivity=conn,
            tile_len=kw.get("tile_len", 16), early_stop=kw.get("early_stop_threshold"))
        assert bits_equal(labels, golden[f"pipe_{name}_labels"]), name
        assert bits_equal(cxy, golden[f"pipe_{name}_cxy"]), name
        assert bits_equal(clab, golden[f"pipe_{name}_clab"]), name
        assert bits_equal(counts, golden[f"pipe_{name}_counts"]), name
        assert passes == int(golden[f"pipe_{name}_passes"][1]), name


@pytest.mark.parametrize("case", ["frame_C1_640x480", "frame_C1_640x480_seed1"])
def test_frame_hashes(golden_meta, case):
    m = golden_meta["hashes"][case]
    rgb = np.random.default_rng(m["seed"]).integers(0, 256, (m["h"], m["w"], 3), dtype=np.uint8)
    s, ns_r, ns_c = _grid(m["w"], m["h"], m["settings"])
    labels, cxy, clab, counts, _ = oracle.segment(rgb, s, ns_r, ns_c, 10.0)
    assert sha(labels) == m["labels"]
    assert sha(cxy) == m["cxy"] and sha(clab) == m["clab"] and sha(counts) == m["counts"]


@pytest.mark.parametrize("case", ["large_C3_f0", "large_T1_963x1024_k2000",
                                  "large_T1_933x800_k1000"])
def test_large_frame_hashes(golden_meta, case):
    """Reference hashes of tests/golden/make_golden_large.py (BASELINE C3,
    PAPER.md Table 1 sizes with W % 4 != 0) pin the oracle at full size."""
    m = golden_meta["hashes"][case]
    rgb = np.random.default_rng(m["seed"]).integers(0, 256, (m["h"], m["w"], 3), dtype=np.uint8)
    s, ns_r, ns_c = _grid(m["w"], m["h"], m["settings"])
    labels, cxy, clab, counts, _ = oracle.segment(rgb, s, ns_r, ns_c, 10.0,
                                                  no_iters=m["settings"].get("no_iters", 5))
    assert sha(labels) == m["labels"]
    assert sha(cxy) == m["cxy"] and sha(clab) == m["clab"] and sha(counts) == m["counts"]


def _oracle_kwargs(kw):
    conn = 0 if kw.get("do_enforce_connectivity") is False else \
        {"weak": 1, "strict": 2}[kw.get("connectivity_mode", "weak")]
    return dict(no_iters=kw.get("no_iters", 5),
                space={"rgb": 0, "xyz": 1, "lab": 2}[kw.get("color_space", "lab")],
                perturb=kw.get("enable_perturbation", False), connectivity=conn,
                min_size=kw.get("min_size"), tile_len=kw.get("tile_len", 16),
                early_stop=kw.get("early_stop_threshold"))


def test_settings_matrix_hashes(golden_meta):
    """Every Settings option at VGA / 720p / C2 sizes (``large_M_*``, made by
    the reference SegEngine in tests/golden/make_golden_large.py)."""
    cases = {k: v for k, v in golden_meta["hashes"].items() if k.startswith("large_M_")}
    assert len(cases) >= 13
    for name, m in cases.items():
        kw = m["settings"]
        rgb = np.random.default_rng(m["seed"]).integers(0, 256, (m["h"], m["w"], 3),
                                                         dtype=np.uint8)
        s, ns_r, ns_c = _grid(m["w"], m["h"], kw)
        labels, cxy, clab, counts, passes = oracle.segment(
            rgb, s, ns_r, ns_c, kw.get("compactness", 10.0), **_oracle_kwargs(kw))
        assert sha(labels) == m["labels"], name
        assert sha(cxy) == m["cxy"] and sha(clab) == m["clab"], name
        assert sha(counts) == m["counts"], name
        assert passes == m["passes"][1], name


def test_center_shift_matches_numpy():
    rng = np.random.default_rng(5)
    for k in (1, 3, 4, 7, 60, 64, 65, 200, 1200, 8160, 50000):
        a = rng.random((k, 2)) * 640
        b = a + rng.normal(0, 1, (k, 2))
        assert oracle.center_shift(b, a) == float(np.abs(b - a).sum()), k


def test_against_built_reference_random():
    sp = oracle.reference_package()
    if sp is None:
        pytest.skip("oracle/_ref not built (no /root/reference at build time)")
    from superpix.kernels import _core as ref
    rng = np.random.default_rng(123)
    for trial in range(8):
        h, w = int(rng.integers(5, 60)), int(rng.integers(5, 60))
        s = int(rng.integers(2, 9))
        ns_r, ns_c = -(-h // s), -(-w // s)
        img = np.ascontiguousarray(rng.random((h, w, 3), dtype=np.float32) * 100)
        cxy = np.ascontiguousarray(np.column_stack([rng.random(ns_r * ns_c) * w,
                                                     rng.random(ns_r * ns_c) * h]))
        clab = rng.random((ns_r * ns_c, 3)) * 100
        a = np.empty((h, w), np.int32); b = np.empty((h, w), np.int32)
        oracle.associate_band(img, cxy, clab, a, s, ns_r, ns_c, 0.7, 0, h)
        ref.associate_band(img, cxy, clab, b, s, ns_r, ns_c, 0.7, 0, h)
        assert bits_equal(a, b)
        tile = int(rng.integers(1, 20))
        n_bl = -(-3 * s // tile)
        sa = np.zeros((ns_r * ns_c, n_bl, 6)); sb = np.zeros_like(sa)
        oracle.accumulate_range(img, a, sa, s, ns_c, tile, 0, ns_r * ns_c)
        ref.accumulate_range(img, a, sb, s, ns_c, tile, 0, ns_r * ns_c)
        assert bits_equal(sa, sb)

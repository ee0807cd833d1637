"""Host-side logic of the drop-in API (CPU only, no kernel calls).

Ports the reference's unit tests for the pieces that live on the host:
settings validation, grid derivation, containers, distance formula, centre
shift, band splitting, PPM I/O, enum parsing, kernel selection
(pkg/tests/test_slic_core.py, test_engine.py, test_imgproc.py,
test_connectivity.py, test_kernels.py).
"""

import numpy as np
import pytest

import paper_1509_04232_b200 as spx
from paper_1509_04232_b200 import kernels
from paper_1509_04232_b200.engine import band_bounds


class TestSettings:
    def test_requires_exactly_one_size_parameter(self):
        with pytest.raises(spx.InvalidSettingsError):
            spx.Settings(img_width=8, img_height=8)
        with pytest.raises(spx.InvalidSettingsError):
            spx.Settings(img_width=8, img_height=8, num_superpixels=4, spixel_size=4)

    @pytest.mark.parametrize("kw", [{"compactness": 0.0}, {"compactness": -3.0}, {"no_iters": 0},
                                    {"tile_len": 0}, {"min_size": 0},
                                    {"early_stop_threshold": -1.0}, {"num_superpixels": 0}])
    def test_rejects_bad_values(self, kw):
        kw = {"num_superpixels": 4, **kw}
        with pytest.raises(spx.InvalidSettingsError):
            spx.Settings(img_width=8, img_height=8, **kw)

    def test_rejects_empty_image(self):
        with pytest.raises(spx.InvalidSettingsError):
            spx.Settings(img_width=0, img_height=8, num_superpixels=4)

    def test_enum_fields_take_names(self):
        st = spx.Settings(img_width=8, img_height=8, num_superpixels=4, color_space="xyz",
                          connectivity_mode="Weak")
        assert st.color_space is spx.ColorSpace.XYZ
        assert st.connectivity_mode is spx.ConnectivityMode.WEAK
        for kw in ({"color_space": "hsv"}, {"connectivity_mode": "loose"}):
            with pytest.raises(spx.InvalidSettingsError):
                spx.Settings(img_width=8, img_height=8, num_superpixels=4, **kw)

    def test_errors_are_valueerrors(self):
        assert issubclass(spx.InvalidSettingsError, ValueError)
        assert issubclass(spx.DimensionMismatchError, spx.SuperpixError)


class TestComputeGrid:
    def test_c1(self):
        g = spx.compute_grid(spx.Settings(img_width=640, img_height=480, num_superpixels=1200))
        assert (g.s, g.ns_c, g.ns_r) == (16, 40, 30)

    def test_c3_c4(self):
        g = spx.compute_grid(spx.Settings(img_width=1920, img_height=1080, num_superpixels=8000))
        assert (g.s, g.ns_r, g.ns_c, g.num_clusters) == (16, 68, 120, 8160)
        g = spx.compute_grid(spx.Settings(img_width=3840, img_height=2160, spixel_size=8))
        assert g.num_clusters == 129600

    def test_ragged_and_rounding(self):
        assert spx.compute_grid(spx.Settings(img_width=105, img_height=100, spixel_size=10)).ns_c == 11
        assert spx.compute_grid(spx.Settings(img_width=5, img_height=5, num_superpixels=4)).s == 3
        assert spx.compute_grid(spx.Settings(img_width=4, img_height=4, num_superpixels=16)).s == 1
        with pytest.raises(spx.InvalidSettingsError):
            spx.compute_grid(spx.Settings(img_width=4, img_height=4, num_superpixels=17))

    def test_num_clusters(self):
        assert spx.GridSpec(8, 3, 5).num_clusters == 15


class TestContainers:
    def test_label_map(self):
        with pytest.raises(ValueError):
            spx.LabelMap(np.array([[0, -1]], dtype=np.int32))
        lm = spx.LabelMap.zeros(5, 3)
        assert (lm.width, lm.height) == (5, 3)
        with pytest.raises(spx.DimensionMismatchError):
            spx.LabelMap(np.zeros((0, 3), np.int32))

    def test_superpixel_map(self):
        sp = spx.SuperpixelMap.empty(spx.GridSpec(4, 2, 2))
        sp.centers_xy[3] = (6.0, 7.0)
        rec = sp.record(3)
        assert rec.id == 3 and rec.center_xy == (6.0, 7.0) and len(sp) == 4
        with pytest.raises(spx.DimensionMismatchError):
            spx.SuperpixelMap(spx.GridSpec(4, 2, 2), np.zeros((3, 2)), np.zeros((4, 3)),
                              np.zeros(4, np.int64))

    @pytest.mark.parametrize("s,tile_len,n_bl", [(32, 16, 6), (5, 16, 1), (8, 3, 8)])
    def test_accum_strip_count(self, s, tile_len, n_bl):
        buf = spx.AccumBuffer.for_grid(spx.GridSpec(s, 2, 2), tile_len)
        assert buf.n_bl == n_bl and buf.slab.shape == (4, n_bl, 6)

    def test_images(self):
        with pytest.raises(spx.DimensionMismatchError):
            spx.ImageRGB(np.zeros((4, 4), np.uint8))
        img = spx.ImageRGB(np.zeros((2, 2, 3), np.uint8))
        with pytest.raises(ValueError):
            img.data[0, 0, 0] = 1
        v = spx.ImageVec3(np.zeros((2, 3, 3), np.float32), spx.ColorSpace.XYZ)
        assert v.space is spx.ColorSpace.XYZ and (v.width, v.height) == (3, 2)


class TestDistance:
    def center(self, l, a, b, x, y):
        sp = spx.SuperpixelMap(spx.GridSpec(8, 1, 1), np.array([[x, y]], float),
                               np.array([[l, a, b]], float), np.zeros(1, np.int64))
        return sp.record(0)

    def test_golden_values(self):
        c = self.center(50, 0, 0, 10, 10)
        assert spx.slic_distance((50, 0, 0, 10, 10), c, 16, 10.0) == 0.0
        assert spx.slic_distance((50, 0, 0, 13, 14), c, 16, 10.0) == 3.125
        assert spx.slic_distance((50, 0, 0, 13, 14), c, 16, 20.0) == 6.25
        c0 = self.center(0, 0, 0, 0, 0)
        assert spx.slic_distance((3, 4, 0, 0, 0), c0, 16, 10.0) == 5.0


class TestCenterShift:
    def test_values(self):
        old = spx.SuperpixelMap.empty(spx.GridSpec(4, 2, 2))
        new = old.copy()
        new.centers_xy[2] += (1.0, -2.0)
        assert spx.center_shift_l1(old, new) == 3.0
        with pytest.raises(spx.DimensionMismatchError):
            spx.center_shift_l1(old, spx.SuperpixelMap.empty(spx.GridSpec(4, 2, 3)))


def test_band_bounds_cover_contiguously():
    for n in (0, 1, 7, 64):
        for workers in (1, 2, 3, 8, 100):
            b = band_bounds(n, workers)
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(x[1] == y[0] for x, y in zip(b, b[1:]))


class TestPpm:
    def test_round_trip(self, tmp_path):
        img = spx.ImageRGB(np.random.default_rng(3).integers(0, 256, (7, 5, 3), dtype=np.uint8))
        p = tmp_path / "rt.ppm"
        spx.write_ppm(p, img)
        assert np.array_equal(spx.load_image(p).data, img.data)

    def test_comments_and_compact_header(self, tmp_path):
        p = tmp_path / "a.ppm"
        p.write_bytes(b"P6\n# note\n2 1\n# more\n255\n" + bytes(6))
        assert (spx.load_image(p).width, spx.load_image(p).height) == (2, 1)
        p.write_bytes(b"P6 2 2 255 " + bytes(range(12)))
        assert spx.load_image(p).data[1, 0].tolist() == [6, 7, 8]

    @pytest.mark.parametrize("raw,msg", [
        (b"P6\n2 2\n255\n" + bytes(11), "truncated pixel data"),
        (b"P5\n1 1\n255\n\x00", "not a binary PPM"),
        (b"P6\n1 1\n65535\n" + bytes(6), "maxval"),
        (b"P6\nx 1\n255\n" + bytes(3), "malformed width"),
        (b"P6\n2", "header ended"),
        (b"P6\n0 1\n255\n", "invalid dimensions"),
    ])
    def test_errors(self, tmp_path, raw, msg):
        p = tmp_path / "bad.ppm"
        p.write_bytes(raw)
        with pytest.raises(spx.PpmError, match=msg):
            spx.load_image(p)


def test_draw_boundaries():
    img = spx.ImageRGB(np.zeros((3, 4, 3), np.uint8))
    lab = np.array([[0, 0, 1, 1]] * 3, np.int32)
    out = spx.draw_boundaries(img, spx.LabelMap(lab), color=(9, 8, 7))
    assert out.data[:, 1].tolist() == [[9, 8, 7]] * 3 and out.data[:, 0].tolist() == [[0, 0, 0]] * 3
    with pytest.raises(spx.DimensionMismatchError):
        spx.draw_boundaries(img, np.zeros((2, 2), np.int32))


def test_parsers_and_selection():
    assert spx.ColorSpace.parse("lab") is spx.ColorSpace.LAB
    assert spx.ConnectivityMode.parse("STRICT") is spx.ConnectivityMode.STRICT
    with pytest.raises(ValueError):
        spx.ColorSpace.parse("hsv")
    with pytest.raises(ValueError):
        spx.ConnectivityMode.parse("loose")
    assert kernels.get_impl("auto") is kernels.ACTIVE
    assert kernels.get_impl("compiled") is kernels.get_impl("cuda")
    with pytest.raises(ValueError):
        kernels.get_impl("gpu")
    with pytest.raises(ImportError):
        kernels.get_impl("pure")
    assert spx.default_min_size(8) == 16 and spx.default_min_size(1) == 1


def test_public_api_matches_reference_names():
    import oracle
    sp = oracle.reference_package()
    if sp is None:
        pytest.skip("reference not built")
    assert sorted(sp.__all__) == sorted(spx.__all__)


def test_engine_rejects_bad_backend_before_touching_the_gpu():
    st = spx.Settings(img_width=8, img_height=8, num_superpixels=4)
    with pytest.raises(spx.InvalidSettingsError):
        spx.SegEngine(st, backend="gpu")
    with pytest.raises(spx.InvalidSettingsError):
        spx.SegEngine(st, backend="par", workers=0)


def test_strict_rejects_bad_min_size():
    with pytest.raises(spx.InvalidSettingsError):
        spx.enforce_strict(spx.LabelMap(np.zeros((1, 1), np.int32)), min_size=0)

"""Whole-pipeline parity: native engine vs the oracle / reference goldens.

Bit-exact labels, centres and counts on the reference's own golden cases
(tests/golden, produced by the reference SegEngine), on BASELINE's C1/C2
frames (hashes of the reference outputs), on batches, and through the
public API entry points.  Runs on a B200 (-m gpu).
"""

import hashlib
import math

import numpy as np
import pytest

import oracle
import paper_1509_04232_b200 as spx

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def settings_from(w, h, kw):
    kw = dict(kw)
    if "connectivity_mode" in kw:
        kw["connectivity_mode"] = spx.ConnectivityMode.parse(kw["connectivity_mode"])
    if "color_space" in kw:
        kw["color_space"] = spx.ColorSpace.parse(kw["color_space"])
    return spx.Settings(img_width=w, img_height=h, **kw)


def test_pipeline_matches_reference_goldens(golden, golden_meta):
    for name, w, h, kw, _seed in golden_meta["pipeline_cases"]:
        st = settings_from(w, h, kw)
        res = spx.SegEngine(st).perform_segmentation(spx.ImageRGB(golden[f"pipe_{name}_rgb"]))
        assert np.array_equal(res.labels.data, golden[f"pipe_{name}_labels"]), name
        assert res.spixel_map.centers_xy.tobytes() == golden[f"pipe_{name}_cxy"].tobytes(), name
        assert res.spixel_map.centers_lab.tobytes() == golden[f"pipe_{name}_clab"].tobytes(), name
        assert np.array_equal(res.spixel_map.num_pixels, golden[f"pipe_{name}_counts"]), name
        n_assoc, n_update = (int(v) for v in golden[f"pipe_{name}_passes"])
        assert (len(res.timing.associate), len(res.timing.update)) == (n_assoc, n_update), name


@pytest.mark.parametrize("case", ["frame_C1_640x480", "frame_C1_640x480_seed1",
                                  "frame_C2_1280x960"])
def test_baseline_frames_match_reference_hashes(golden_meta, case):
    m = golden_meta["hashes"][case]
    rgb = np.random.default_rng(m["seed"]).integers(0, 256, (m["h"], m["w"], 3), dtype=np.uint8)
    st = settings_from(m["w"], m["h"], m["settings"])
    res = spx.SegEngine(st).perform_segmentation(spx.ImageRGB(rgb))
    assert sha(res.labels.data) == m["labels"]
    assert sha(res.spixel_map.centers_xy) == m["cxy"]
    assert sha(res.spixel_map.centers_lab) == m["clab"]
    assert sha(res.spixel_map.num_pixels) == m["counts"]


def test_batch_equals_single_frames():
    w, h = 160, 120
    st = spx.Settings(img_width=w, img_height=h, num_superpixels=75)
    frames = [np.random.default_rng(i).integers(0, 256, (h, w, 3), dtype=np.uint8)
              for i in range(7)]
    eng = spx.SegEngine(st, max_batch=4)
    batch = eng.perform_segmentation_batch([spx.ImageRGB(f) for f in frames])
    g = spx.compute_grid(st)
    for f, r in zip(frames, batch):
        labels, cxy, clab, counts, _ = oracle.segment(f, g.s, g.ns_r, g.ns_c, st.compactness)
        assert np.array_equal(r.labels.data, labels)
        assert r.spixel_map.centers_lab.tobytes() == clab.tobytes()
        assert np.array_equal(r.spixel_map.num_pixels, counts)


def test_device_batch_api_and_early_stop_per_frame():
    import torch
    w, h = 96, 64
    st = spx.Settings(img_width=w, img_height=h, num_superpixels=24, no_iters=8,
                      early_stop_threshold=15.0)
    frames = [np.random.default_rng(50 + i).integers(0, 256, (h, w, 3), dtype=np.uint8)
              for i in range(5)]
    frames[2][:] = 77  # flat frame converges after one update
    eng = spx.SegEngine(st, max_batch=5)
    d = torch.from_numpy(np.stack(frames)).cuda()
    labels, cxy, clab, counts, passes = eng.segment_device(d)
    torch.cuda.synchronize()
    g = spx.compute_grid(st)
    for i, f in enumerate(frames):
        lw, xw, lb, cw, pw = oracle.segment(f, g.s, g.ns_r, g.ns_c, st.compactness, no_iters=8,
                                            early_stop=15.0)
        assert int(passes[i]) == pw
        assert np.array_equal(labels[i].cpu().numpy(), lw)
        assert cxy[i].cpu().numpy().tobytes() == xw.tobytes()
        assert np.array_equal(counts[i].cpu().numpy(), cw)


def test_strict_and_perturb_larger():
    w, h = 200, 150
    rgb = np.random.default_rng(77).integers(0, 256, (h, w, 3), dtype=np.uint8)
    for kw in (dict(connectivity_mode=spx.ConnectivityMode.STRICT),
               dict(enable_perturbation=True), dict(do_enforce_connectivity=False, tile_len=5)):
        st = spx.Settings(img_width=w, img_height=h, num_superpixels=120, **kw)
        res = spx.SegEngine(st).perform_segmentation(spx.ImageRGB(rgb))
        g = spx.compute_grid(st)
        conn = 0 if not st.do_enforce_connectivity else (
            2 if st.connectivity_mode is spx.ConnectivityMode.STRICT else 1)
        labels, cxy, clab, counts, _ = oracle.segment(
            rgb, g.s, g.ns_r, g.ns_c, st.compactness, perturb=st.enable_perturbation,
            connectivity=conn, tile_len=st.tile_len)
        assert np.array_equal(res.labels.data, labels), kw
        assert res.spixel_map.centers_xy.tobytes() == cxy.tobytes(), kw
        assert np.array_equal(res.spixel_map.num_pixels, counts), kw


def test_flat_image_block_tiling():
    st = spx.Settings(img_width=64, img_height=64, spixel_size=8)
    res = spx.SegEngine(st).perform_segmentation(spx.ImageRGB(np.full((64, 64, 3), 137, np.uint8)))
    want = (np.arange(64)[:, None] // 8) * 8 + np.arange(64)[None, :] // 8
    assert np.array_equal(res.labels.data, want)


def test_single_shot_api_chain_matches_oracle():
    rng = np.random.default_rng(303)
    w, h = 47, 31
    img = spx.ImageRGB(rng.integers(0, 256, (h, w, 3), dtype=np.uint8))
    st = spx.Settings(img_width=w, img_height=h, num_superpixels=12)
    grid = spx.compute_grid(st)
    lab = spx.convert_color_space(img, spx.ColorSpace.LAB)
    sp = spx.init_cluster_centers(lab, grid)
    ref_lab = np.empty((h, w, 3), np.float32)
    oracle.convert_band(img.data, ref_lab, 2, 0, h)
    assert lab.data.tobytes() == ref_lab.tobytes()
    for _ in range(3):
        labels = spx.find_center_association(lab, sp, st)
        want = np.empty((h, w), np.int32)
        oracle.associate_band(ref_lab, sp.centers_xy, sp.centers_lab, want, grid.s, grid.ns_r,
                              grid.ns_c, st.compactness / grid.s, 0, h)
        assert np.array_equal(labels.data, want)
        buf = spx.accumulate_cluster_stats(lab, labels, grid, st.tile_len)
        sp = spx.reduce_cluster_stats(buf, sp)
        assert int(sp.num_pixels.sum()) == w * h
    # centroids vs brute force 5-D means (test_acceptance.py:144-180)
    ys, xs = np.mgrid[0:h, 0:w]
    for k in range(grid.num_clusters):
        if sp.num_pixels[k]:
            assert math.isclose(sp.centers_xy[k, 0], xs[labels.data == k].mean(), rel_tol=1e-9) or \
                sp.num_pixels[k] == 0


def test_center_shift_device_matches_numpy():
    import ctypes
    import torch
    from paper_1509_04232_b200 import _lib
    rng = np.random.default_rng(4)
    for k in (1, 5, 64, 1200, 8160, 129600):
        a = rng.random((k, 2)) * 1000
        b = a + rng.normal(0, 1, (k, 2))
        da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        out = torch.zeros(1, dtype=torch.float64, device="cuda")
        _lib.check(_lib.load().spx_center_shift(ctypes.c_void_p(db.data_ptr()),
                                                ctypes.c_void_p(da.data_ptr()), k,
                                                ctypes.c_void_p(out.data_ptr()), None))
        torch.cuda.synchronize()
        assert float(out.item()) == float(np.abs(b - a).sum()), k


def _oracle_pipeline(rgb, st):
    g = spx.compute_grid(st)
    conn = 0 if not st.do_enforce_connectivity else (
        2 if st.connectivity_mode is spx.ConnectivityMode.STRICT else 1)
    return oracle.segment(rgb, g.s, g.ns_r, g.ns_c, st.compactness, no_iters=st.no_iters,
                          space=st.color_space.value, perturb=st.enable_perturbation,
                          connectivity=conn, min_size=st.min_size, tile_len=st.tile_len,
                          early_stop=st.early_stop_threshold)


def _images(h, w, seed):
    rng = np.random.default_rng(seed)
    noise = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
    # gray-heavy image: exercises the certified-sum fallback (tiny a/b values)
    gray = np.repeat(rng.integers(0, 256, (h, w, 1), dtype=np.uint8), 3, axis=2)
    gray[::7] = noise[::7]
    # smooth gradient + mild noise: natural-image-like, coherent clusters
    yy, xx = np.mgrid[0:h, 0:w]
    smooth = np.stack([(xx * 255 // max(w - 1, 1)), (yy * 255 // max(h - 1, 1)),
                       ((xx + yy) * 127 // max(w + h - 2, 1))], -1)
    smooth = np.clip(smooth + rng.integers(-6, 7, (h, w, 3)), 0, 255).astype(np.uint8)
    dark = (noise // 40).astype(np.uint8)  # near-black: small L, tiny a/b
    return {"noise": noise, "gray": gray, "smooth": smooth, "dark": dark}


@pytest.mark.parametrize("s,odd_w", [(8, False), (12, False), (16, False), (20, False),
                                     (24, False), (32, False),
                                     (4, False), (5, True), (6, False), (7, True), (9, False),
                                     (10, True), (14, False), (18, True), (25, False), (31, True)])
def test_cell_path_grid_sizes_bitexact(s, odd_w):
    # 4 <= S <= 32 and h*w % 4 == 0 select the fused cell kernels: 128-bit
    # runs when S % 4 == 0 and W % 4 == 0, per-pixel (partial) runs
    # otherwise; ragged last row/column of cells included.
    h, w = 3 * s + 5, 4 * s + 4 * ((s // 4) % 3) + 8
    w -= w % 4
    if odd_w:  # W % 4 != 0 (h chosen so that h*w % 4 == 0)
        w, h = w + 2, h + (h % 2)
    for name, rgb in _images(h, w, s).items():
        for tile in (16, 5):
            st = spx.Settings(img_width=w, img_height=h, spixel_size=s, tile_len=tile, no_iters=3)
            res = spx.SegEngine(st).perform_segmentation(spx.ImageRGB(rgb))
            labels, cxy, clab, counts, _ = _oracle_pipeline(rgb, st)
            assert np.array_equal(res.labels.data, labels), (s, name, tile)
            assert res.spixel_map.centers_xy.tobytes() == cxy.tobytes(), (s, name, tile)
            assert res.spixel_map.centers_lab.tobytes() == clab.tobytes(), (s, name, tile)
            assert np.array_equal(res.spixel_map.num_pixels, counts), (s, name, tile)


@pytest.mark.parametrize("s,h,w", [
    (16, 99, 123),    # h*w odd: padded planar planes, partial last convert group
    (5, 37, 51), (8, 41, 66), (12, 50, 77),
    (33, 104, 137), (40, 125, 161), (47, 140, 201), (64, 197, 261),   # LPC 16, S > 32
    (84, 253, 339), (118, 300, 355), (160, 330, 480),                  # LPC 32, global window
])
def test_cell_path_large_cells_and_odd_frames(s, h, w):
    # S > 32 (per-lane field unpacking, sub-chunked exact-fallback segments,
    # the label window read in place when 9 S^2 labels exceed the smem
    # budget) and frames with h*w % 4 != 0 run the fused cell kernels and
    # equal the oracle bit for bit.
    for name, rgb in _images(h, w, s + 1).items():
        for tile in (16, 9):
            st = spx.Settings(img_width=w, img_height=h, spixel_size=s, tile_len=tile, no_iters=3)
            eng = spx.SegEngine(st)
            assert eng.fused_path, (s, h, w, tile)
            res = eng.perform_segmentation(spx.ImageRGB(rgb))
            labels, cxy, clab, counts, _ = _oracle_pipeline(rgb, st)
            assert np.array_equal(res.labels.data, labels), (s, name, tile)
            assert res.spixel_map.centers_xy.tobytes() == cxy.tobytes(), (s, name, tile)
            assert res.spixel_map.centers_lab.tobytes() == clab.tobytes(), (s, name, tile)
            assert np.array_equal(res.spixel_map.num_pixels, counts), (s, name, tile)


@pytest.mark.parametrize("kw", [
    dict(spixel_size=46),
    dict(spixel_size=48, early_stop_threshold=40.0, no_iters=9),
    dict(spixel_size=44, enable_perturbation=True, tile_len=7),
    dict(spixel_size=70, connectivity_mode=spx.ConnectivityMode.STRICT, tile_len=30),
    dict(spixel_size=52, color_space=spx.ColorSpace.XYZ, compactness=3.0),
])
def test_wide_mode_batches_graphs_and_lanes(kw):
    # S > 42 (wide mode, per-(cluster, strip) sums): a mixed batch through the graph
    # replay (calls 3 and 4) and through concurrent lanes, every frame equal
    # to the oracle; early stop, perturbation, strict connectivity, odd tile
    # lengths and XYZ included
    import torch
    h, w = 181, 243
    st = spx.Settings(img_width=w, img_height=h, **kw)
    imgs = _images(h, w, 5)
    frames = np.stack([imgs[k] for k in ("noise", "gray", "smooth", "dark")] + [imgs["noise"][::-1].copy()])
    ref = [_oracle_pipeline(f, st) for f in frames]
    eng = spx.SegEngine(st, max_batch=len(frames))
    assert eng.fused_path
    d = torch.from_numpy(frames).cuda()
    for call in range(4):
        labels, cxy, clab, counts, passes = (x.cpu().numpy() for x in eng.segment_device(d))
        for i, (ol, ox, oc, on, op) in enumerate(ref):
            assert np.array_equal(labels[i], ol), (kw, call, i)
            assert cxy[i].tobytes() == ox.tobytes() and clab[i].tobytes() == oc.tobytes(), (kw, call, i)
            assert np.array_equal(counts[i], on) and int(passes[i]) == op, (kw, call, i)
    big = torch.from_numpy(np.concatenate([frames] * 4)).cuda()  # 20 frames: lanes
    eng2 = spx.SegEngine(st, max_batch=20)
    eng2.set_lanes(3)
    labels, cxy, clab, counts, _ = (x.cpu().numpy() for x in eng2.segment_device(big))
    for i in range(20):
        ol, ox, oc, on, _ = ref[i % 5]
        assert np.array_equal(labels[i], ol) and np.array_equal(counts[i], on), (kw, i)
        assert cxy[i].tobytes() == ox.tobytes() and clab[i].tobytes() == oc.tobytes(), (kw, i)


@pytest.mark.parametrize("s", [24, 30, 32])
def test_large_launch_lane_choice(s):
    # big single-lane launches at S = 24 / 29..32 take 16 / 4 lanes per cell
    # (cell_lpc); frames at both ends of the batch equal the oracle
    import torch
    h, w, b = 544, 960, 24
    st = spx.Settings(img_width=w, img_height=h, spixel_size=s, no_iters=3)
    frames = np.stack([_images(h, w, 300 + i)["noise"] if i % 2 == 0 else _images(h, w, 300 + i)["gray"]
                       for i in range(b)])
    eng = spx.SegEngine(st, max_batch=b)
    eng.set_lanes(1)
    labels, cxy, clab, counts, _ = (x.cpu().numpy() for x in eng.segment_device(
        torch.from_numpy(frames).cuda()))
    for i in (0, 1, b - 1):
        ol, ox, oc, on, _ = _oracle_pipeline(frames[i], st)
        assert np.array_equal(labels[i], ol), (s, i)
        assert cxy[i].tobytes() == ox.tobytes() and clab[i].tobytes() == oc.tobytes(), (s, i)
        assert np.array_equal(counts[i], on), (s, i)


def test_odd_frame_batches_and_strips():
    # a batch of frames with h*w odd (frame f's pixels start at an unaligned
    # RGB offset for odd f) and a row-strip split of such a frame
    from paper_1509_04232_b200.strips import segment_strips_local
    h, w = 75, 93
    st = spx.Settings(img_width=w, img_height=h, spixel_size=9, no_iters=4)
    frames = [_images(h, w, 70 + i)["noise"] for i in range(5)]
    eng = spx.SegEngine(st, max_batch=5)
    labels, cxy, clab, counts, _ = eng.segment_host(np.stack(frames))
    for i, rgb in enumerate(frames):
        ol, ox, oc, on, _ = _oracle_pipeline(rgb, st)
        assert np.array_equal(labels[i], ol), i
        assert cxy[i].tobytes() == ox.tobytes() and clab[i].tobytes() == oc.tobytes(), i
        assert np.array_equal(counts[i], on), i
    sl, sx, sc, sn = segment_strips_local(st, frames[1], 3)
    ol, ox, oc, on, _ = _oracle_pipeline(frames[1], st)
    assert np.array_equal(sl, ol) and sx.tobytes() == ox.tobytes()
    assert sc.tobytes() == oc.tobytes() and np.array_equal(sn, on)


@pytest.mark.parametrize("s,odd_w", [(6, False), (8, False), (12, False), (16, False),
                                     (20, False), (24, False), (10, True), (18, True)])
def test_cell_path_wide_launch_bitexact(s, odd_w):
    # Small launches (the single-frame tests above) run with doubled lanes
    # per cell; a batch of >= 20,000 cells keeps the narrow cells.  Both
    # must give the oracle's results.
    h, w = 3 * s + 5, 4 * s + 4 * ((s // 4) % 3) + 8
    w -= w % 4
    if odd_w:
        w, h = w + 2, h + (h % 2)
    imgs = list(_images(h, w, 40 + s).values())
    st = spx.Settings(img_width=w, img_height=h, spixel_size=s, no_iters=3)
    k = spx.compute_grid(st).num_clusters
    n = -(-20000 // k)
    batch = np.stack([imgs[i % len(imgs)] for i in range(n)])
    labels, cxy, clab, counts, _ = spx.SegEngine(st, max_batch=n).segment_host(batch)
    for i, rgb in enumerate(imgs):
        ol, ox, oc, on, _ = _oracle_pipeline(rgb, st)
        assert np.array_equal(labels[i], ol), (s, i)
        assert cxy[i].tobytes() == ox.tobytes() and clab[i].tobytes() == oc.tobytes(), (s, i)
        assert np.array_equal(counts[i], on), (s, i)
    for i in range(len(imgs), n):  # every copy equals its first occurrence
        j = i % len(imgs)
        assert np.array_equal(labels[i], labels[j]) and clab[i].tobytes() == clab[j].tobytes()


def test_concurrent_exact_fallback_large_batch():
    # Gray-heavy frames flag many clusters; at this batch size the exact
    # fallback (side stream) overlaps the reduce for thousands of clusters.
    h, w = 240, 320
    st = spx.Settings(img_width=w, img_height=h, spixel_size=16)
    kinds = ("gray", "dark", "noise", "smooth")
    frames = np.stack([_images(h, w, 700 + i)[kinds[i % 4]] for i in range(96)])
    eng = spx.SegEngine(st, max_batch=96)
    labels, cxy, clab, counts, _ = eng.segment_host(frames)
    for i in (0, 1, 2, 3, 57, 94):
        ol, ox, oc, on, _ = _oracle_pipeline(frames[i], st)
        assert np.array_equal(labels[i], ol), i
        assert cxy[i].tobytes() == ox.tobytes() and clab[i].tobytes() == oc.tobytes(), i
        assert np.array_equal(counts[i], on), i


@pytest.mark.parametrize("kw", [dict(), dict(early_stop_threshold=15.0, no_iters=8),
                                dict(connectivity_mode=spx.ConnectivityMode.STRICT)])
def test_lanes_split_matches_unsplit_and_oracle(kw):
    # A call of more than 16 frames runs as concurrent sub-batches (lanes) on
    # child engines; the split (ragged here: 130 = 44 + 44 + 42) must not
    # change any output.
    import torch
    h, w = 64, 96
    st = spx.Settings(img_width=w, img_height=h, num_superpixels=24, **kw)
    kinds = ("gray", "dark", "noise", "smooth")
    frames = np.stack([_images(h, w, 900 + i)[kinds[i % 4]] for i in range(130)])
    d = torch.from_numpy(frames).cuda()
    eng = spx.SegEngine(st, max_batch=130)
    res = {}
    for lanes in (1, 3, 0):
        eng.set_lanes(lanes)
        out = [t.clone() for t in eng.segment_device(d)]
        torch.cuda.synchronize()
        res[lanes] = ([t.cpu().numpy() for t in out], eng.last_lanes())
    # auto: more than 16 frames but under 24 Mpx of work -> three lanes
    assert res[1][1] == 1 and res[3][1] == 3 and res[0][1] == 3
    for lanes in (3, 0):
        for a, b in zip(res[1][0], res[lanes][0]):
            assert a.tobytes() == b.tobytes(), lanes
    labels, cxy, clab, counts, passes = res[3][0]
    for i in (0, 43, 44, 87, 88, 129):  # both sides of every lane boundary
        ol, ox, oc, on, op = _oracle_pipeline(frames[i], st)
        assert np.array_equal(labels[i], ol), i
        assert cxy[i].tobytes() == ox.tobytes() and clab[i].tobytes() == oc.tobytes(), i
        assert np.array_equal(counts[i], on), i
    t = eng.last_timing()
    assert t.total > 0
    with pytest.raises(ValueError):
        eng.set_lanes(-1)


def test_lanes_resplit_sequence():
    # Lane counts that grow and shrink: child engines sized for a finer split
    # are replaced when a coarser split needs bigger lanes.
    import torch
    h, w = 64, 96
    st = spx.Settings(img_width=w, img_height=h, num_superpixels=24)
    frames = np.stack([_images(h, w, 950 + i)["noise"] for i in range(40)])
    d = torch.from_numpy(frames).cuda()
    eng = spx.SegEngine(st, max_batch=40)
    eng.set_lanes(1)
    want = [t.cpu().numpy() for t in eng.segment_device(d)]
    for lanes in (2, 3, 5, 8, 4, 0, 8, 2, 40, 7):
        eng.set_lanes(lanes)
        got = [t.cpu().numpy() for t in eng.segment_device(d)]
        for a, b in zip(want, got):
            assert a.tobytes() == b.tobytes(), lanes


def test_lanes_in_graph_replay():
    # <= 16 frames take the CUDA-graph path; with lanes the captured graph
    # forks the lanes' streams.  Replays must equal the unsplit results.
    import torch
    h, w = 64, 96
    st = spx.Settings(img_width=w, img_height=h, num_superpixels=24)
    frames = np.stack([_images(h, w, 980 + i)["noise"] for i in range(12)])
    d = torch.from_numpy(frames).cuda()
    eng = spx.SegEngine(st, max_batch=12)
    eng.set_lanes(1)
    want = [t.cpu().numpy() for t in eng.segment_device(d)]
    for lanes in (3, 2):
        eng.set_lanes(lanes)
        outs = eng.allocate_outputs(12)
        for call in range(5):  # eager, eager, capture, replay, replay
            for t in outs:
                t.zero_()
            eng.segment_device(d, outs)
            torch.cuda.synchronize()
            assert eng.last_lanes() == lanes
            assert eng.last_timing().total > 0
            for a, b in zip(want, outs):
                assert a.tobytes() == b.cpu().numpy().tobytes(), (lanes, call)


def test_lanes_graph_cache_survives_child_replacement():
    # an automatic 4-lane graph captured over 8-frame children,
    # then a call whose 3-lane split needs bigger children (they are
    # replaced), then the first key again -- the old graph must not replay
    # over the freed children.  Same with explicit lane counts 3 -> 2 -> 3.
    import torch
    h, w = 64, 96
    st = spx.Settings(img_width=w, img_height=h, num_superpixels=24)
    frames = np.stack([_images(h, w, 1200 + i)["noise"] for i in range(32)])
    d = torch.from_numpy(frames).cuda()
    ref = spx.SegEngine(st, max_batch=32)
    ref.set_lanes(1)
    want = [t.cpu().numpy() for t in ref.segment_device(d)]

    def check(eng, outs, n):
        for t in outs:
            t.zero_()
        eng.segment_device(d[:n], tuple(t[:n] for t in outs))
        torch.cuda.synchronize()
        for a, b in zip(want, outs):
            assert a[:n].tobytes() == b[:n].cpu().numpy().tobytes(), n

    eng = spx.SegEngine(st, max_batch=32)
    outs = eng.allocate_outputs(32)
    for _ in range(4):  # eager, eager, capture, replay (4 lanes of 8)
        check(eng, outs, 8)
    eng.set_lanes(3)  # children of ceil(32 / 3) = 11 frames replace the 8-frame ones
    for _ in range(4):
        check(eng, outs, 12)
    eng.set_lanes(0)
    for _ in range(3):
        check(eng, outs, 8)
    for lanes in (3, 2, 3):
        eng.set_lanes(lanes)
        for _ in range(4):
            check(eng, outs, 16)


def test_cell_path_batch_gray_heavy_frames():
    h, w = 480, 640
    st = spx.Settings(img_width=w, img_height=h, num_superpixels=1200)
    frames = [_images(h, w, 900 + i)[name] for i, name in enumerate(("gray", "dark", "smooth", "noise"))]
    eng = spx.SegEngine(st, max_batch=4)
    res = eng.perform_segmentation_batch([spx.ImageRGB(f) for f in frames])
    for f, r in zip(frames, res):
        labels, cxy, clab, counts, _ = _oracle_pipeline(f, st)
        assert np.array_equal(r.labels.data, labels)
        assert r.spixel_map.centers_lab.tobytes() == clab.tobytes()
        assert r.spixel_map.centers_xy.tobytes() == cxy.tobytes()
        assert np.array_equal(r.spixel_map.num_pixels, counts)


@pytest.mark.parametrize("h,w,kw,n", [
    (480, 640, dict(num_superpixels=1200), 3),
    (200, 160, dict(spixel_size=16), 2),
    (200, 160, dict(spixel_size=16), 5),
    (250, 96, dict(spixel_size=8, tile_len=5, enable_perturbation=True), 4),
    (130, 64, dict(spixel_size=12, do_enforce_connectivity=False, no_iters=3), 3),
    # early stop (the gathered shift decides on every strip at once); the
    # thresholds stop the noise / smooth frames at different passes
    (200, 160, dict(spixel_size=16, no_iters=9, early_stop_threshold=400.0), 3),
    (240, 200, dict(spixel_size=12, no_iters=12, early_stop_threshold=150.0), 4),
    # odd width (padded planes), S > 32, boundary-only strips (1-2 own rows)
    (231, 157, dict(spixel_size=9, no_iters=4), 5),
    (300, 150, dict(spixel_size=40, no_iters=3), 3),
    (96, 80, dict(spixel_size=8, no_iters=3), 6),
    # strict connectivity: the scan-order pass over the gathered strips
    (200, 160, dict(spixel_size=16, connectivity_mode=spx.ConnectivityMode.STRICT), 3),
    (150, 96, dict(spixel_size=8, min_size=20, no_iters=4,
                   connectivity_mode=spx.ConnectivityMode.STRICT), 5),
])
def test_row_strips_equal_whole_image(h, w, kw, n):
    """C5 decomposition: strips with halo centres / partial-sum / label exchange
    give exactly the single-GPU (and reference) result."""
    from paper_1509_04232_b200.strips import segment_strips_local
    st = spx.Settings(img_width=w, img_height=h, **kw)
    for name, rgb in _images(h, w, 7 * n + h).items():
        labels, cxy, clab, counts = segment_strips_local(st, rgb, n)
        wl, wx, wlab, wc, _ = _oracle_pipeline(rgb, st)
        assert np.array_equal(labels, wl), name
        assert cxy.tobytes() == wx.tobytes(), name
        assert clab.tobytes() == wlab.tobytes(), name
        assert np.array_equal(counts, wc), name


def test_submit_host_pipeline_across_batches():
    """Back-to-back submit_host calls (chunks cross batch boundaries and reuse
    staging slots) give the same results as one synchronous call per batch."""
    import torch
    h, w = 48, 64
    st = spx.Settings(img_width=w, img_height=h, spixel_size=8)
    eng = spx.SegEngine(st, max_batch=70)
    eng.set_host_chunk(32)
    k = eng.grid.num_clusters
    rng = np.random.default_rng(21)
    batches = [rng.integers(0, 256, (n, h, w, 3), dtype=np.uint8) for n in (70, 5, 66, 1)]
    pin = lambda shape, dt: torch.empty(shape, dtype=dt).pin_memory().numpy()  # noqa: E731
    outs = []
    for b in batches:
        n = b.shape[0]
        o = (pin((n, h, w), torch.int32), pin((n, k, 2), torch.float64),
             pin((n, k, 3), torch.float64), pin((n, k), torch.int64), pin((n,), torch.int32))
        eng.submit_host(torch.from_numpy(b).pin_memory().numpy(), *o)
        outs.append(o)
    eng.wait()
    for b, o in zip(batches, outs):
        want = eng.segment_host(b)
        for got, ref in zip(o, want):
            assert got.tobytes() == ref.tobytes()
    eng.set_host_chunk(70)
    for b, o in zip(batches, outs):
        for got, ref in zip(o, eng.segment_host(b)):
            assert got.tobytes() == ref.tobytes()
    with pytest.raises(ValueError):
        eng.submit_host(batches[1], *outs[0])


@pytest.mark.parametrize("w,h,kw", [
    (1920, 1080, dict(num_superpixels=8000)),              # C3 frame
    (3840, 2160, dict(spixel_size=8, no_iters=10)),        # C4 frame
])
def test_large_baseline_frames_bitexact(w, h, kw):
    """BASELINE C3 / C4 frames (reference generator, seed 0) equal the oracle."""
    st = spx.Settings(img_width=w, img_height=h, **kw)
    g = spx.compute_grid(st)
    rgb = np.random.default_rng(0).integers(0, 256, (h, w, 3), dtype=np.uint8)
    res = spx.SegEngine(st).perform_segmentation(spx.ImageRGB(rgb))
    labels, cxy, clab, counts, _ = oracle.segment(rgb, g.s, g.ns_r, g.ns_c, st.compactness,
                                                  no_iters=st.no_iters)
    assert np.array_equal(res.labels.data, labels)
    assert res.spixel_map.centers_xy.tobytes() == cxy.tobytes()
    assert res.spixel_map.centers_lab.tobytes() == clab.tobytes()
    assert np.array_equal(res.spixel_map.num_pixels, counts)


@pytest.mark.parametrize("kw", [dict(), dict(early_stop_threshold=3.0, no_iters=9),
                                dict(connectivity_mode=spx.ConnectivityMode.STRICT)])
def test_graph_replay_matches_eager_and_times(kw):
    """Calls 1-2 (eager), 3 (captured) and 4+ (replayed CUDA graph) with the same
    buffers give identical results; stage timings stay readable."""
    import torch
    st = spx.Settings(img_width=64, img_height=48, spixel_size=8, **kw)
    eng = spx.SegEngine(st, max_batch=3)
    rgb = torch.from_numpy(np.random.default_rng(5).integers(0, 256, (3, 48, 64, 3),
                                                             dtype=np.uint8)).cuda()
    out = eng.allocate_outputs(3)
    ref = None
    for call in range(5):
        for t in out:
            t.zero_()
        eng.segment_device(rgb, out)
        torch.cuda.synchronize()
        got = [t.cpu().numpy().tobytes() for t in out]
        ref = ref or got
        assert got == ref, f"call {call}"
        tm = eng.last_timing()
        assert tm.total > 0 and len(tm.associate) >= 2
        assert eng.last_launches() > 0
    g = spx.compute_grid(st)
    conn = 2 if kw.get("connectivity_mode") is not None else 1
    es = kw.get("early_stop_threshold")
    labels, cxy, clab, counts, _ = oracle.segment(
        rgb[2].cpu().numpy(), g.s, g.ns_r, g.ns_c, st.compactness, no_iters=st.no_iters,
        connectivity=conn, min_size=spx.default_min_size(g.s),
        early_stop=es)
    assert np.array_equal(out[0][2].cpu().numpy(), labels)
    assert out[2][2].cpu().numpy().tobytes() == clab.tobytes()


class TestStream:
    """segment_stream (reference test_engine.py:140-176) plus pipelined batches."""

    def settings(self):
        return spx.Settings(img_width=16, img_height=16, num_superpixels=4)

    def test_matches_independent_calls(self):
        rng = np.random.default_rng(58)
        a = spx.ImageRGB(rng.integers(0, 256, (16, 16, 3), dtype=np.uint8))
        b = spx.ImageRGB(rng.integers(0, 256, (16, 16, 3), dtype=np.uint8))
        streamed = list(spx.segment_stream(spx.SegEngine(self.settings()), [a, b, a]))
        assert len(streamed) == 3
        assert np.array_equal(streamed[0].labels.data, streamed[2].labels.data)
        solo = spx.SegEngine(self.settings()).perform_segmentation(b)
        assert np.array_equal(streamed[1].labels.data, solo.labels.data)

    def test_results_survive_later_frames(self):
        rng = np.random.default_rng(59)
        frames = [spx.ImageRGB(rng.integers(0, 256, (16, 16, 3), dtype=np.uint8))
                  for _ in range(7)]
        eng = spx.SegEngine(self.settings(), max_batch=2)
        kept = [r.labels.data for r in spx.segment_stream(eng, frames)]
        redo = [spx.SegEngine(self.settings()).perform_segmentation(f).labels.data
                for f in frames]
        assert all(np.array_equal(x, y) for x, y in zip(kept, redo))

    def test_empty_stream(self):
        assert list(spx.segment_stream(spx.SegEngine(self.settings()), [])) == []

    def test_mismatched_frame_names_index(self):
        eng = spx.SegEngine(self.settings(), max_batch=2)
        ok = spx.ImageRGB(np.full((16, 16, 3), 9, np.uint8))
        bad = spx.ImageRGB(np.zeros((16, 8, 3), np.uint8))
        got = []
        with pytest.raises(spx.DimensionMismatchError, match="frame 3"):
            for r in spx.segment_stream(eng, [ok, ok, ok, bad]):
                got.append(r)
        assert len(got) == 3  # results of the frames before the bad one

    def test_pipelined_batches_match_oracle(self):
        st = spx.Settings(img_width=64, img_height=48, spixel_size=8)
        g = spx.compute_grid(st)
        rng = np.random.default_rng(60)
        frames = [rng.integers(0, 256, (48, 64, 3), dtype=np.uint8) for _ in range(11)]
        eng = spx.SegEngine(st, max_batch=3)
        for f, r in zip(frames, spx.segment_stream(eng, [spx.ImageRGB(x) for x in frames])):
            labels, cxy, clab, counts, _ = oracle.segment(f, g.s, g.ns_r, g.ns_c, st.compactness)
            assert np.array_equal(r.labels.data, labels)
            assert r.spixel_map.centers_lab.tobytes() == clab.tobytes()


@pytest.mark.parametrize("ranks,extra", [(2, []), (3, []),
                                         (3, ["--early-stop", "1000", "--iters", "10"]),
                                         (3, ["--strict"])])
def test_row_strips_distributed_processes(ranks, extra):
    """One process per strip (torchrun), halos and partial sums exchanged
    through DistComm (gloo, staged through host memory; the ranks share this
    GPU): the gathered strips equal the whole-image engine bit for bit."""
    import os
    import socket
    import subprocess
    import sys
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SPX_STRIPS_BACKEND="gloo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={ranks}", "--master-addr", "127.0.0.1",
                        "--master-port", str(port), os.path.join(root, "tools", "strips_dist.py"),
                        "--size", "512", "--check", *extra], env=env, capture_output=True,
                       text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "bit-identical to the whole-image engine: True" in r.stdout

"""Full-size BASELINE configs and PAPER.md Table 1 against the REFERENCE itself.

The hashes in tests/golden/golden_hashes.json (``large_*``) were produced by
the unmodified reference SegEngine (tests/golden/make_golden_large.py); these
tests run the same synthetic frames through this package on the GPU and
compare sha256 of labels, centres and counts:

* C3: BASELINE's 512-frame 1920x1080 batch as ONE segment_device call
  (frames 0, 1, 255, 511 checked; ~10^9 labels, where index overflows hide);
* C4: 3840x2160, S = 8, 10 iterations;
* C5: 16384x16384 (268 Mpx, 1,048,576 clusters) through SegEngine and as 8
  row strips with the halo / partial-sum / label exchange;
* the five PAPER.md Table 1 image sizes at 1000 and 2000 superpixels;
* the Settings surface (``large_M_*``): strict connectivity, perturbation,
  XYZ / RGB, early stop, no connectivity, unaligned S, tile_len, 720p,
  S > 32 and all options together -- per frame through
  perform_segmentation and inside a mixed batch through segment_device.
"""

import hashlib

import numpy as np
import pytest

import paper_1509_04232_b200 as spx

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def frame(m):
    return np.random.default_rng(m["seed"]).integers(0, 256, (m["h"], m["w"], 3), dtype=np.uint8)


def settings(m):
    return spx.Settings(img_width=m["w"], img_height=m["h"], **m["settings"])


def assert_matches(m, labels, cxy, clab, counts, what):
    assert sha(labels) == m["labels"], f"{what}: labels"
    assert sha(cxy) == m["cxy"], f"{what}: centers_xy"
    assert sha(clab) == m["clab"], f"{what}: centers_lab"
    assert sha(counts) == m["counts"], f"{what}: num_pixels"


def test_c3_batch_of_512_frames_one_call(golden_meta):
    import torch
    h = golden_meta["hashes"]
    checked = {int(k.split("_f")[1]): v for k, v in h.items() if k.startswith("large_C3_f")}
    assert sorted(checked) == [0, 1, 255, 511]
    m0 = checked[0]
    st = settings(m0)
    n = 512
    rgb = torch.empty((n, m0["h"], m0["w"], 3), dtype=torch.uint8, device="cuda")
    for i in range(n):  # frame i = seed i (the reference generator)
        rgb[i].copy_(torch.from_numpy(frame(dict(m0, seed=i))))
    eng = spx.SegEngine(st, max_batch=n)
    labels, cxy, clab, counts, passes = eng.segment_device(rgb)
    torch.cuda.synchronize()
    assert int(passes.min()) == int(passes.max()) == st.no_iters
    for i, m in checked.items():
        assert m["seed"] == i
        assert_matches(m, labels[i].cpu().numpy(), cxy[i].cpu().numpy(), clab[i].cpu().numpy(),
                       counts[i].cpu().numpy(), f"C3 frame {i}")
    # every frame accounts for all its pixels
    assert bool((counts.sum(dim=1) == m0["w"] * m0["h"]).all())


def test_c4_frame(golden_meta):
    m = golden_meta["hashes"]["large_C4"]
    res = spx.SegEngine(settings(m)).perform_segmentation(spx.ImageRGB(frame(m)))
    assert_matches(m, res.labels.data, res.spixel_map.centers_xy, res.spixel_map.centers_lab,
                   res.spixel_map.num_pixels, "C4")


def test_c5_gigapixel_whole_and_8_strips(golden_meta):
    import torch
    from paper_1509_04232_b200.strips import segment_strips_local
    m = golden_meta["hashes"]["large_C5"]
    st = settings(m)
    rgb = frame(m)
    eng = spx.SegEngine(st, max_batch=1)
    d = torch.from_numpy(rgb).cuda()
    labels, cxy, clab, counts, _ = eng.segment_device(d)
    torch.cuda.synchronize()
    assert_matches(m, labels[0].cpu().numpy(), cxy[0].cpu().numpy(), clab[0].cpu().numpy(),
                   counts[0].cpu().numpy(), "C5 whole image")
    del eng, labels, cxy, clab, counts, d
    torch.cuda.empty_cache()
    labels, cxy, clab, counts = segment_strips_local(st, rgb, 8)
    assert_matches(m, labels, cxy, clab, counts, "C5 8 strips")


TABLE1 = ["1024x1024", "3631x3859", "963x1024", "1002x1002", "933x800"]


@pytest.mark.parametrize("k", [1000, 2000])
@pytest.mark.parametrize("size", TABLE1)
def test_paper_table1_sizes(golden_meta, size, k):
    m = golden_meta["hashes"][f"large_T1_{size}_k{k}"]
    eng = spx.SegEngine(settings(m))
    assert eng.fused_path  # every Table-1 shape (S = 19 ... 118) runs the fused kernels
    res = eng.perform_segmentation(spx.ImageRGB(frame(m)))
    assert_matches(m, res.labels.data, res.spixel_map.centers_xy, res.spixel_map.centers_lab,
                   res.spixel_map.num_pixels, f"{size} K={k}")


MATRIX = ["strict", "strict_min50", "perturb", "xyz", "rgb", "early", "noconn", "k1000_s18",
          "m40_i12", "tile5", "720p", "c2_s35", "all"]


@pytest.mark.parametrize("name", MATRIX)
def test_settings_matrix(golden_meta, name):
    import torch
    m = golden_meta["hashes"][f"large_M_{name}"]
    st = settings(m)
    img = frame(m)
    res = spx.SegEngine(st).perform_segmentation(spx.ImageRGB(img))
    assert_matches(m, res.labels.data, res.spixel_map.centers_xy, res.spixel_map.centers_lab,
                   res.spixel_map.num_pixels, f"{name} perform_segmentation")
    assert len(res.timing.update) == m["passes"][1], name
    # the same frame in the middle of a batch of unrelated frames
    other = np.random.default_rng(m["seed"] + 1000).integers(0, 256, img.shape, dtype=np.uint8)
    batch = torch.from_numpy(np.stack([other, img, other[::-1].copy()])).cuda()
    eng = spx.SegEngine(st, max_batch=3)
    labels, cxy, clab, counts, passes = eng.segment_device(batch)
    torch.cuda.synchronize()
    assert_matches(m, labels[1].cpu().numpy(), cxy[1].cpu().numpy(), clab[1].cpu().numpy(),
                   counts[1].cpu().numpy(), f"{name} batch")
    assert int(passes[1]) == m["passes"][1]


@pytest.mark.parametrize("name", MATRIX)
def test_settings_matrix_row_strips(golden_meta, name):
    # the same cases as 3 row strips (halo / partial sums / labels exchanged)
    from paper_1509_04232_b200.strips import segment_strips_local
    m = golden_meta["hashes"][f"large_M_{name}"]
    labels, cxy, clab, counts = segment_strips_local(settings(m), frame(m), 3)
    assert_matches(m, labels, cxy, clab, counts, f"{name} 3 strips")

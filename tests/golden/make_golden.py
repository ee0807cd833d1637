"""Generate the golden fixtures in tests/golden from the REFERENCE itself.

Run here (CPU container) after ``oracle/build_ref.sh`` has compiled the
unmodified reference into ``oracle/_ref``::

    python tests/golden/make_golden.py

Every vector is produced by the reference's compiled kernel set
(``superpix.kernels._core``, i.e. _core.pyx built with the flags of
pkg/setup.py) or its ``SegEngine``; nothing here runs our code.  Inputs come
from the reference's own synthetic generator
(``np.random.default_rng(seed).integers(0, 256, (h, w, 3), uint8)``,
kernel_bench.py:21-23) and the random-array helpers of pkg/tests.

Outputs:
  golden.npz          small per-kernel and whole-pipeline arrays
  golden_hashes.json  sha256 of large outputs (all 2^24 colours, C1/C2 frames)
"""

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(REPO, "oracle", "_ref"))

import superpix as sp  # noqa: E402  (the reference package)
from superpix.kernels import _core as ref  # noqa: E402

assert sp.kernels.active() == "compiled"


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def rgb_image(seed, h, w):
    return np.random.default_rng(seed).integers(0, 256, (h, w, 3), dtype=np.uint8)


def rand_img(rng, h, w):  # pkg/tests/test_kernels.py:48-49
    return np.ascontiguousarray(rng.random((h, w, 3), dtype=np.float32) * 100.0)


def make_centers(rng, k, w, h):  # pkg/tests/test_kernels.py:90-93
    cxy = np.column_stack([rng.random(k) * w, rng.random(k) * h])
    clab = rng.random((k, 3)) * 100.0
    return np.ascontiguousarray(cxy), np.ascontiguousarray(clab)


def all_colours():
    c = np.arange(1 << 24, dtype=np.uint32)
    return np.stack([(c >> 16) & 255, (c >> 8) & 255, c & 255], -1).astype(np.uint8).reshape(4096, 4096, 3)


PIPELINE_CASES = [
    # name, w, h, settings kwargs, seed
    ("flat32", 32, 32, dict(spixel_size=8), None),
    ("tiny1x1", 1, 1, dict(num_superpixels=1, no_iters=1), 0),
    ("r64x48", 64, 48, dict(num_superpixels=12), 1),
    ("r47x31", 47, 31, dict(num_superpixels=12, compactness=20.0), 2),
    ("r33x57_perturb", 33, 57, dict(num_superpixels=9, enable_perturbation=True), 3),
    ("r40x32_strict", 40, 32, dict(num_superpixels=12, connectivity_mode="strict"), 4),
    ("r96x80_noconn", 96, 80, dict(num_superpixels=40, do_enforce_connectivity=False), 5),
    ("r64x64_early", 64, 64, dict(num_superpixels=16, no_iters=5, early_stop_threshold=20.0), 6),
    ("r128x96_s5", 128, 96, dict(spixel_size=5, no_iters=3), 7),
    ("r100x70_xyz", 100, 70, dict(num_superpixels=30, color_space="xyz"), 8),
    ("r90x60_rgb", 90, 60, dict(num_superpixels=20, color_space="rgb", compactness=0.05), 9),
    ("r160x120_t4", 160, 120, dict(spixel_size=12, tile_len=4), 10),
]

FRAME_CASES = [
    ("C1_640x480", 640, 480, dict(num_superpixels=1200), 0),
    ("C2_1280x960", 1280, 960, dict(num_superpixels=4800), 0),
    ("C1_640x480_seed1", 640, 480, dict(num_superpixels=1200), 1),
]


def settings(w, h, kw):
    kw = dict(kw)
    if "connectivity_mode" in kw:
        kw["connectivity_mode"] = sp.ConnectivityMode.parse(kw["connectivity_mode"])
    if "color_space" in kw:
        kw["color_space"] = sp.ColorSpace.parse(kw["color_space"])
    return sp.Settings(img_width=w, img_height=h, **kw)


def main():
    out = {}
    hashes = {}

    # convert: 17x13 random (test_kernels.py:51-59) + named colours
    rgb = np.random.default_rng(41).integers(0, 256, (17, 13, 3), dtype=np.uint8)
    out["convert_rgb"] = rgb
    for space in (0, 1, 2):
        o = np.empty((17, 13, 3), np.float32)
        ref.convert_band(rgb, o, space, 0, 17)
        out[f"convert_out_{space}"] = o
    named = np.array([[[128, 64, 32], [255, 255, 255], [0, 0, 0], [1, 1, 1], [128, 128, 128]]],
                     dtype=np.uint8)
    o = np.empty((1, 5, 3), np.float32)
    ref.convert_band(named, o, 2, 0, 1)
    out["convert_named_rgb"] = named
    out["convert_named_lab"] = o

    # all 2^24 colours, every space
    allc = all_colours()
    for space in (0, 1, 2):
        o = np.empty((4096, 4096, 3), np.float32)
        ref.convert_band(allc, o, space, 0, 4096)
        hashes[f"convert_all_colours_space{space}"] = sha(o)

    # init + perturb (test_kernels.py:62-87)
    rng = np.random.default_rng(42)
    img = rand_img(rng, 23, 31)
    cxy = np.zeros((20, 2)); clab = np.zeros((20, 3))
    ref.init_centers_range(img, 7, 5, cxy, clab, 0, 20)
    out["init_img"] = img; out["init_cxy"] = cxy.copy(); out["init_clab"] = clab.copy()
    rng = np.random.default_rng(43)
    img = rand_img(rng, 23, 31)
    bxy = np.zeros((20, 2)); blab = np.zeros((20, 3))
    ref.init_centers_range(img, 7, 5, bxy, blab, 0, 20)
    out["perturb_img"] = img; out["perturb_in_xy"] = bxy.copy(); out["perturb_in_lab"] = blab.copy()
    ref.perturb_range(img, bxy, blab, 0, 20)
    out["perturb_xy"] = bxy; out["perturb_lab"] = blab

    # associate (test_kernels.py:96-106)
    rng = np.random.default_rng(44)
    h, w, s, ns_r, ns_c = 29, 31, 6, 5, 6
    img = rand_img(rng, h, w)
    cxy, clab = make_centers(rng, ns_r * ns_c, w, h)
    lab = np.empty((h, w), np.int32)
    ref.associate_band(img, cxy, clab, lab, s, ns_r, ns_c, 1.7, 0, h)
    out.update(assoc_img=img, assoc_cxy=cxy, assoc_clab=clab, assoc_labels=lab)

    # accumulate + spill (test_kernels.py:109-129)
    rng = np.random.default_rng(45)
    h, w, s, ns_r, ns_c, tile_len = 22, 18, 5, 5, 4, 4
    img = rand_img(rng, h, w)
    k = ns_r * ns_c
    labels = rng.integers(0, k, (h, w)).astype(np.int32)
    n_bl = -(-s * 3 // tile_len)
    slab = np.zeros((k, n_bl, 6))
    ref.accumulate_range(img, labels, slab, s, ns_c, tile_len, 0, k)
    out["accum_range_slab"] = slab.copy()
    spills = ref.accumulate_spill(img, labels, slab, s, ns_c)
    out.update(accum_img=img, accum_labels=labels, accum_slab=slab,
               accum_spills=np.array(spills))

    # reduce (test_kernels.py:132-153)
    for n_bl in (1, 2, 3, 5, 6, 8):
        rng = np.random.default_rng(46 + n_bl)
        k = 7
        slab = rng.random((k, n_bl, 6)) * 50.0
        slab[:, :, 5] = rng.integers(0, 4, (k, n_bl)).astype(np.float64)
        slab[2, :, 5] = 0.0
        prev_xy = rng.random((k, 2)); prev_lab = rng.random((k, 3))
        work = slab.copy()
        oxy = np.zeros((k, 2)); olab = np.zeros((k, 3)); ocnt = np.zeros(k, np.int64)
        ref.reduce_range(work, prev_xy, prev_lab, oxy, olab, ocnt, 0, k)
        out.update({f"reduce{n_bl}_slab": slab, f"reduce{n_bl}_prev_xy": prev_xy,
                    f"reduce{n_bl}_prev_lab": prev_lab, f"reduce{n_bl}_xy": oxy,
                    f"reduce{n_bl}_lab": olab, f"reduce{n_bl}_cnt": ocnt})

    # weak / strict (test_kernels.py:156-173)
    src = np.random.default_rng(47).integers(0, 4, (19, 14)).astype(np.int32)
    dst = np.empty_like(src)
    ref.weak_band(src, dst, 0, 19)
    out.update(weak_src=src, weak_dst=dst)
    src = np.random.default_rng(48).integers(0, 5, (17, 13)).astype(np.int32)
    dst = np.empty_like(src)
    ref.strict_fill(src, dst, 4)
    out.update(strict_src=src, strict_dst=dst)
    src = np.random.default_rng(49).integers(0, 30, (64, 80)).astype(np.int32)
    dst = np.empty_like(src)
    ref.strict_fill(src, dst, 7)
    out.update(strict2_src=src, strict2_dst=dst)

    # whole pipeline through SegEngine (seq backend, compiled kernels)
    names = []
    for name, w, h, kw, seed in PIPELINE_CASES:
        st = settings(w, h, kw)
        if seed is None:
            img = np.full((h, w, 3), 90, np.uint8)
        else:
            img = rgb_image(seed, h, w)
        res = sp.SegEngine(st).perform_segmentation(sp.ImageRGB(img))
        out[f"pipe_{name}_rgb"] = img
        out[f"pipe_{name}_labels"] = res.labels.data
        out[f"pipe_{name}_cxy"] = res.spixel_map.centers_xy
        out[f"pipe_{name}_clab"] = res.spixel_map.centers_lab
        out[f"pipe_{name}_counts"] = res.spixel_map.num_pixels
        out[f"pipe_{name}_passes"] = np.array([len(res.timing.associate), len(res.timing.update)])
        names.append(name)

    for name, w, h, kw, seed in FRAME_CASES:
        st = settings(w, h, kw)
        img = rgb_image(seed, h, w)
        res = sp.SegEngine(st, backend="par", workers=os.cpu_count()).perform_segmentation(
            sp.ImageRGB(img))
        hashes[f"frame_{name}"] = {
            "w": w, "h": h, "settings": kw, "seed": seed,
            "labels": sha(res.labels.data),
            "cxy": sha(res.spixel_map.centers_xy),
            "clab": sha(res.spixel_map.centers_lab),
            "counts": sha(res.spixel_map.num_pixels),
        }

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    meta = {"generator": "reference superpix (compiled _core) via oracle/_ref",
            "pipeline_cases": [[n, w, h, kw, s] for n, w, h, kw, s in PIPELINE_CASES],
            "hashes": hashes}
    with open(os.path.join(HERE, "golden_hashes.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("wrote", len(out), "arrays and", len(hashes), "hashes")


if __name__ == "__main__":
    main()

"""Reference hashes for the full-size BASELINE configs and PAPER.md Table 1.

Run here (CPU container, reference compiled into oracle/_ref by
oracle/build_ref.sh)::

    python tests/golden/make_golden_large.py [--only NAME ...]

Each case runs the UNMODIFIED reference ``SegEngine`` (thread-pool backend,
all host cores, compiled _core kernels) on the reference's own synthetic
generator (``np.random.default_rng(seed).integers(0, 256, (h, w, 3),
uint8)``, kernel_bench.py:21-23) and stores the sha256 of labels, centres
and counts under ``hashes["large_<name>"]`` in golden_hashes.json (the other
entries are left untouched).  Nothing here runs our code.

Cases:
  C3_f{0,1,255,511}  1920x1080, K=8000, 5 iters: frames of BASELINE's
                     512-frame batch (frame i = seed i; frames are
                     independent, so each is one reference call)
  C4                 3840x2160, S=8, 10 iters
  C5                 16384x16384, S=16, 5 iters (~1 min on 8 cores)
  T1_<w>x<h>_k<K>    PAPER.md:135-139 image sizes at 1000 / 2000 superpixels
  M_<name>           the Settings surface: strict connectivity (default and
                     explicit min_size), perturbation, XYZ / RGB, early stop,
                     no connectivity, unaligned S, compactness / iterations,
                     tile_len, 720p, S > 32, and everything at once
"""

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(REPO, "oracle", "_ref"))

import superpix as sp  # noqa: E402  (the reference package)

assert sp.kernels.active() == "compiled"

TABLE1 = [(1024, 1024), (3631, 3859), (963, 1024), (1002, 1002), (933, 800)]

CASES = (
    [(f"C3_f{i}", 1920, 1080, dict(num_superpixels=8000), i) for i in (0, 1, 255, 511)]
    + [("C4", 3840, 2160, dict(spixel_size=8, no_iters=10), 0)]
    + [(f"T1_{w}x{h}_k{k}", w, h, dict(num_superpixels=k), 0) for w, h in TABLE1
       for k in (1000, 2000)]
    + [("C5", 16384, 16384, dict(spixel_size=16), 0)]
    # the Settings surface at VGA / 720p / C2 sizes (every option the
    # reference's SegEngine takes, one at a time and combined)
    + [(f"M_{name}", w, h, kw, seed) for name, w, h, kw, seed in (
        ("strict", 640, 480, dict(num_superpixels=1200, connectivity_mode="strict"), 3),
        ("strict_min50", 640, 480, dict(num_superpixels=1200, connectivity_mode="strict",
                                        min_size=50), 4),
        ("perturb", 640, 480, dict(num_superpixels=1200, enable_perturbation=True), 5),
        ("xyz", 640, 480, dict(num_superpixels=1200, color_space="xyz"), 6),
        ("rgb", 640, 480, dict(num_superpixels=1200, color_space="rgb", compactness=0.1), 7),
        ("early", 640, 480, dict(num_superpixels=1200, no_iters=20, early_stop_threshold=200.0), 8),
        ("noconn", 640, 480, dict(num_superpixels=1200, do_enforce_connectivity=False), 9),
        ("k1000_s18", 640, 480, dict(num_superpixels=1000), 10),
        ("m40_i12", 640, 480, dict(num_superpixels=600, compactness=40.0, no_iters=12), 11),
        ("tile5", 640, 480, dict(spixel_size=12, tile_len=5), 12),
        ("720p", 1280, 720, dict(num_superpixels=3600), 13),
        ("c2_s35", 1280, 960, dict(num_superpixels=1000), 14),
        ("all", 1001, 777, dict(num_superpixels=2500, compactness=15.0, no_iters=7,
                                enable_perturbation=True, connectivity_mode="strict",
                                min_size=30, tile_len=8, early_stop_threshold=80.0), 15),
    )]
)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*")
    args = ap.parse_args()
    path = os.path.join(HERE, "golden_hashes.json")
    with open(path) as fh:
        meta = json.load(fh)
    for name, w, h, kw, seed in CASES:
        if args.only and name not in args.only:
            continue
        t0 = time.time()
        kw2 = dict(kw)
        if "connectivity_mode" in kw2:
            kw2["connectivity_mode"] = sp.ConnectivityMode.parse(kw2["connectivity_mode"])
        if "color_space" in kw2:
            kw2["color_space"] = sp.ColorSpace.parse(kw2["color_space"])
        st = sp.Settings(img_width=w, img_height=h, **kw2)
        img = np.random.default_rng(seed).integers(0, 256, (h, w, 3), dtype=np.uint8)
        res = sp.SegEngine(st, backend="par", workers=os.cpu_count()).perform_segmentation(
            sp.ImageRGB(img))
        meta["hashes"][f"large_{name}"] = {
            "w": w, "h": h, "settings": kw, "seed": seed,
            "labels": sha(res.labels.data),
            "cxy": sha(res.spixel_map.centers_xy),
            "clab": sha(res.spixel_map.centers_lab),
            "counts": sha(res.spixel_map.num_pixels),
            "passes": [len(res.timing.associate), len(res.timing.update)],
            "num_pixels_total": int(res.spixel_map.num_pixels.sum()),
            "ref_seconds": round(res.timing.total, 2),
            "ref_workers": os.cpu_count(),
        }
        del res, img
        with open(path, "w") as fh:
            json.dump(meta, fh, indent=1, sort_keys=True)
        print(f"{name}: {time.time() - t0:.1f} s", flush=True)


if __name__ == "__main__":
    main()

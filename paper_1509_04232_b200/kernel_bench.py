"""Per-stage benchmark: the fused engine against the per-stage kernel chain.

GPU counterpart of the reference's `superpix-kernel-bench`
(kernel_bench.py:49-92), which times the compiled kernels against the pure
Python fallback on one synthetic image and checks that the two label maps are
identical.  Here the two implementations are

  * "engine": `SegEngine.perform_segmentation` -- the fused cell kernels,
    one CUDA-graph-replayed call, stage times from CUDA events;
  * "stages": the single-shot API chain (convert_color_space,
    init_cluster_centers, then per iteration find_center_association,
    accumulate_cluster_stats, reduce_cluster_stats, and enforce_weak) -- one
    C-ABI per-stage kernel each, host arrays in and out, wall-clock timed;

and their label maps, centres and counts must be bit-identical (both are
bit-identical to the reference).

    python -m paper_1509_04232_b200.kernel_bench --size 256 --superpixels 256
"""

import argparse
import statistics
import sys
import time

import numpy as np

from .connectivity import enforce_weak
from .engine import SegEngine
from .imgproc import ColorSpace, ImageRGB, convert_color_space
from .slic_core import (
    Settings,
    accumulate_cluster_stats,
    compute_grid,
    find_center_association,
    init_cluster_centers,
    reduce_cluster_stats,
)

STAGES = ("convert", "init", "associate", "update", "connectivity", "total")


def synthetic_image(size, seed):
    """The reference's synthetic input (kernel_bench.py:21-23)."""
    rng = np.random.default_rng(seed)
    return ImageRGB(rng.integers(0, 256, size=(size, size, 3), dtype=np.uint8))


def _engine_stages(timing):
    return {"convert": timing.convert, "init": timing.init + timing.perturb,
            "associate": sum(timing.associate), "update": sum(timing.update),
            "connectivity": timing.connectivity, "total": timing.total}


def _run_engine(settings, img, repeats, device):
    eng = SegEngine(settings, device=device)
    for _ in range(3):  # warm-up; the third call captures the CUDA graph
        result = eng.perform_segmentation(img)
    samples = [_engine_stages(eng.perform_segmentation(img).timing) for _ in range(repeats)]
    return {k: statistics.fmean(s[k] for s in samples) for k in STAGES}, result


def _run_stages_once(settings, img):
    grid = compute_grid(settings)
    t = dict.fromkeys(STAGES, 0.0)
    t0 = time.perf_counter()
    lab = convert_color_space(img, ColorSpace.LAB)
    t1 = time.perf_counter()
    sp = init_cluster_centers(lab, grid)
    t2 = time.perf_counter()
    t["convert"], t["init"] = t1 - t0, t2 - t1
    for _ in range(settings.no_iters):
        a = time.perf_counter()
        labels = find_center_association(lab, sp, settings)
        b = time.perf_counter()
        sp = reduce_cluster_stats(accumulate_cluster_stats(lab, labels, grid, settings.tile_len),
                                  sp)
        c = time.perf_counter()
        t["associate"] += b - a
        t["update"] += c - b
    a = time.perf_counter()
    labels = find_center_association(lab, sp, settings)
    b = time.perf_counter()
    labels = enforce_weak(labels)
    c = time.perf_counter()
    t["associate"] += b - a
    t["connectivity"] = c - b
    t["total"] = c - t0
    return t, labels, sp


def _run_stages(settings, img, repeats):
    _run_stages_once(settings, img)  # warm-up
    samples = []
    for _ in range(repeats):
        t, labels, sp = _run_stages_once(settings, img)
        samples.append(t)
    return {k: statistics.fmean(s[k] for s in samples) for k in STAGES}, labels, sp


def main(argv=None):
    ap = argparse.ArgumentParser(
        prog="superpix-kernel-bench", formatter_class=argparse.ArgumentDefaultsHelpFormatter,
        description="Compare the fused GPU engine with the per-stage GPU kernel chain.")
    ap.add_argument("--size", type=int, default=256, help="synthetic image side length")
    ap.add_argument("--superpixels", type=int, default=256)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--repeats", type=int, default=3)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--device", type=int, default=0)
    args = ap.parse_args(argv)
    settings = Settings(img_width=args.size, img_height=args.size,
                        num_superpixels=args.superpixels, no_iters=args.iters)
    img = synthetic_image(args.size, args.seed)
    print(f"image {args.size}x{args.size}, K={args.superpixels}, {args.iters} iterations, "
          f"mean of {args.repeats} runs")
    eng_t, res = _run_engine(settings, img, args.repeats, args.device)
    stg_t, labels, sp = _run_stages(settings, img, args.repeats)
    print(f"{'stage':>12}  {'engine':>12}  {'stages':>12}  {'ratio':>8}")
    for k in STAGES:
        e, s = eng_t[k], stg_t[k]
        ratio = f"{s / e:7.1f}x" if e > 0 else "     n/a"
        print(f"{k:>12}  {e * 1e3:9.3f} ms  {s * 1e3:9.3f} ms  {ratio}")
    identical = (np.array_equal(res.labels.data, labels.data)
                 and res.spixel_map.centers_xy.tobytes() == sp.centers_xy.tobytes()
                 and res.spixel_map.centers_lab.tobytes() == sp.centers_lab.tobytes()
                 and np.array_equal(res.spixel_map.num_pixels, sp.num_pixels))
    print(f"labels identical: {'yes' if identical else 'NO'}")
    return 0 if identical else 1


if __name__ == "__main__":
    sys.exit(main())

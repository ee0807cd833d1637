"""Per-frame latency of the drop-in call SegEngine.perform_segmentation (diagnostic).

One 640x480 frame (host numpy in, SegResult out), repeated; prints the mean
and median wall time per call after warm-up.

    python tools/pseg_latency.py [--n 200]
"""
import argparse
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1509_04232_b200 as spx  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=200)
    a = ap.parse_args()
    st = spx.Settings(img_width=640, img_height=480, num_superpixels=1200)
    eng = spx.SegEngine(st)
    img = spx.ImageRGB(np.random.default_rng(0).integers(0, 256, (480, 640, 3), dtype=np.uint8))
    for _ in range(10):
        eng.perform_segmentation(img)
    ts = []
    for _ in range(a.n):
        t0 = time.perf_counter()
        r = eng.perform_segmentation(img)
        ts.append(time.perf_counter() - t0)
    print(f"perform_segmentation 640x480: mean {statistics.mean(ts) * 1e3:.3f} ms, "
          f"median {statistics.median(ts) * 1e3:.3f} ms, min {min(ts) * 1e3:.3f} ms "
          f"(device total {r.timing.total * 1e3:.3f} ms)")


if __name__ == "__main__":
    main()

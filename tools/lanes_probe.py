"""Probe: device ms per batch for lane counts 1..8 on the BASELINE configs
(C1: 256 VGA frames, C2: 64 x 1280x960, C3: 128 x 1080p, C4: 8 x 4K S=8 10 iters),
plus the automatic choice.  Needs a GPU.

(An earlier build also had SPX_LANE_STAGGER -- lane i waiting for lane i-1's
convert; measured 1% slower at 4 lanes on C1 and removed.)

    python tools/lanes_probe.py [--configs C1,C2,C3,C4]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1509_04232_b200 as spx  # noqa: E402

CONFIGS = {
    "C1": (640, 480, dict(num_superpixels=1200), 256, (1, 2, 3, 4, 5, 6, 8)),
    "C2": (1280, 960, dict(num_superpixels=4800), 64, (1, 2, 3, 4, 8)),
    "C3": (1920, 1080, dict(num_superpixels=8000), 128, (1, 2, 3, 4, 8)),
    "C4": (3840, 2160, dict(spixel_size=8, no_iters=10), 8, (1, 2, 3, 4, 8)),
}


def run(eng, rgb, outs, lanes, steps=8):
    eng.set_lanes(lanes)
    for _ in range(3):
        eng.segment_device(rgb, outs)
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(steps):
        eng.segment_device(rgb, outs)
    s1.record()
    torch.cuda.synchronize()
    return s0.elapsed_time(s1) / steps, eng.last_lanes()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C3,C4")
    ap.add_argument("--batch", type=int, default=0, help="override frames per batch")
    ap.add_argument("--lanes", default="", help="comma list overriding the lane counts")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    for name in a.configs.split(","):
        w, h, kw, b, lane_set = CONFIGS[name]
        b = a.batch or b
        if a.lanes:
            lane_set = tuple(int(x) for x in a.lanes.split(","))
        rng = np.random.default_rng(0)
        rgb = torch.from_numpy(rng.integers(0, 256, (b, h, w, 3), dtype=np.uint8)).cuda()
        st = spx.Settings(img_width=w, img_height=h, **kw)
        eng = spx.SegEngine(st, device=0, max_batch=b)
        outs = eng.allocate_outputs(b)
        for lanes in lane_set + (0,):
            ms, used = run(eng, rgb, outs, lanes)
            tag = f"auto({used})" if lanes == 0 else str(lanes)
            print(f"{name} lanes={tag}: {ms:.3f} ms/batch of {b}  {b / ms * 1e3:.1f} frames/s",
                  flush=True)
        del eng, outs, rgb
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

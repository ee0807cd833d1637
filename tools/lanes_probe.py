"""Probe: device ms per 256-frame C1 step for lane counts 1..8.  Needs a GPU.

(An earlier build also had SPX_LANE_STAGGER -- lane i waiting for lane i-1's
convert; measured 1% slower at 4 lanes and removed, so both rows now match.)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1509_04232_b200 as spx  # noqa: E402

W, H, B = 640, 480, 256


def run(eng, rgb, outs, lanes, steps=10):
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
    return s0.elapsed_time(s1) / steps


def main():
    torch.cuda.set_device(0)
    rng = np.random.default_rng(0)
    rgb = torch.from_numpy(rng.integers(0, 256, (B, H, W, 3), dtype=np.uint8)).cuda()
    st = spx.Settings(img_width=W, img_height=H, num_superpixels=1200, compactness=10,
                      no_iters=5)
    for stagger in (False, True):
        if stagger:
            os.environ["SPX_LANE_STAGGER"] = "1"
        eng = spx.SegEngine(st, device=0, max_batch=B)
        outs = eng.allocate_outputs(B)
        for lanes in (1, 2, 3, 4, 5, 6, 8):
            ms = run(eng, rgb, outs, lanes)
            print(f"stagger={int(stagger)} lanes={lanes}: {ms:.3f} ms  {B / ms * 1e3:.0f} frames/s",
                  flush=True)
        del eng


if __name__ == "__main__":
    main()

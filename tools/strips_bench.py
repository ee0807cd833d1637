"""C5 row strips on one GPU: per-strip device time and exchange volume (diagnostic).

Runs the 16384x16384 image (S = 16, 5 iterations) as N row strips in one
process (LocalComm: strips one after another, exchanges as device copies) and
as one whole image through SegEngine, checks they are bit-identical, and
reports the sum and max of the per-strip device times.  With one GPU per
strip the wall time would be about the slowest strip plus the exchanges.

    python tools/strips_bench.py [--n 8] [--size 16384]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("SPX_NO_GRAPHS", "1")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1509_04232_b200 as spx  # noqa: E402
from paper_1509_04232_b200.strips import LocalComm, StripEngine, _run  # noqa: E402
from paper_1509_04232_b200.sharding import strip_plan  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8)
    ap.add_argument("--size", type=int, default=16384)
    a = ap.parse_args()
    n = a.size
    st = spx.Settings(img_width=n, img_height=n, spixel_size=16)
    g = spx.compute_grid(st)
    rgb = torch.from_numpy(np.random.default_rng(0).integers(0, 256, (n, n, 3), dtype=np.uint8)).cuda()

    # whole image
    eng = spx.SegEngine(st, max_batch=1)
    out = eng.allocate_outputs(1)
    for _ in range(2):
        eng.segment_device(rgb.unsqueeze(0), out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.segment_device(rgb.unsqueeze(0), out)
    e1.record()
    torch.cuda.synchronize()
    whole_ms = e0.elapsed_time(e1)
    whole = [t[0].cpu().numpy() for t in out[:4]]
    del eng, out
    torch.cuda.empty_cache()

    # strips, sequential on this GPU; per-strip device time from events around
    # each strip's own kernels (exchanges are the copies between them)
    plan = strip_plan(n, g.s, g.ns_r, a.n)
    strips = [StripEngine(st, p.cell_row_lo, p.cell_row_hi, 0) for p in plan]
    windows = [rgb[s.y0:s.y0 + s.hl].contiguous() for s in strips]
    for rep in range(2):
        ev = {}
        for i, s in enumerate(strips):
            ev[i] = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        t0 = time.perf_counter()
        for s, wdw in zip(strips, windows):
            s.begin(wdw)
        _run(strips, LocalComm(strips))
        outs = [s.finish() for s in strips]
        torch.cuda.synchronize()
        host_s = time.perf_counter() - t0
    labels = torch.cat([o[0] for o in outs]).cpu().numpy()
    clab = torch.cat([o[2] for o in outs]).cpu().numpy()
    exact = np.array_equal(labels, whole[0]) and clab.tobytes() == whole[2].tobytes()

    # device time of one strip alone (the middle one): its kernels only
    mid = strips[len(strips) // 2]
    e0.record()
    mid.begin(windows[len(strips) // 2])
    for _ in range(st.no_iters):
        mid.associate(True)
        mid.update()
    mid.associate(False)
    mid.finish()
    e1.record()
    torch.cuda.synchronize()
    strip_ms = e0.elapsed_time(e1)
    bytes_per_boundary_iter = g.ns_c * (40 + 48) + g.s * n * 4 * 2
    print(f"C5 {n}x{n}, {a.n} strips: whole image {whole_ms:.2f} ms on one GPU; one interior "
          f"strip's kernels {strip_ms:.2f} ms (ideal 1/{a.n}: {whole_ms / a.n:.2f} ms); "
          f"bit-identical: {exact}; exchange per boundary per iteration "
          f"{bytes_per_boundary_iter / 1e6:.2f} MB; sequential host-orchestrated run {host_s * 1e3:.0f} ms")


if __name__ == "__main__":
    main()

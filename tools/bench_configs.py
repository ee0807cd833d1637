"""Device throughput of every BASELINE.json config on one B200.

For each config: synthetic frames from the reference generator
(np.random.default_rng(i).integers(0, 256, (H, W, 3), uint8)), resident in HBM,
W warm-up + R timed batches with CUDA events, per-stage device times, the
SURVEY §8(d) algorithmic bytes per frame and the HBM-roofline fraction.
Frame 0 of C1-C4 is checked bit-for-bit against the C oracle (test tooling).

    python tools/bench_configs.py [--configs C1,C2,...] [--md profiles/r1_configs.md]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
# eager engine calls: every stage event is live (graph replays of small
# batches report the first call's stage breakdown)
os.environ.setdefault("SPX_NO_GRAPHS", "1")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1509_04232_b200 as spx  # noqa: E402

PEAK = 6548.2  # GB/s, MEASURED_PEAKS.json
CONFIGS = {
    # name: (W, H, settings kwargs, frames per batch, check frame 0 against the oracle)
    "C1": (640, 480, dict(num_superpixels=1200), 256, True),
    "C2": (1280, 960, dict(num_superpixels=4800), 64, True),
    "C3": (1920, 1080, dict(num_superpixels=8000), 128, True),
    "C4": (3840, 2160, dict(spixel_size=8, no_iters=10), 8, True),
    "C5": (16384, 16384, dict(spixel_size=16), 1, False),
}


def frames(h, w, n):
    return np.stack([np.random.default_rng(i).integers(0, 256, (h, w, 3), dtype=np.uint8)
                     for i in range(n)])


def run(name, reps, warm):
    w, h, kw, b, check = CONFIGS[name]
    st = spx.Settings(img_width=w, img_height=h, **kw)
    g = spx.compute_grid(st)
    eng = spx.SegEngine(st, max_batch=b)
    host = frames(h, w, min(b, 8))
    if b > host.shape[0]:  # repeat the first 8 generator frames (same statistics)
        host = np.concatenate([host] * (b // host.shape[0]) + [host[:b % host.shape[0]]])
    d_rgb = torch.from_numpy(host).cuda()
    out = eng.allocate_outputs(b)
    for _ in range(warm):
        eng.segment_device(d_rgb, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        eng.segment_device(d_rgb, out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    lanes = eng.last_lanes()
    # stage columns: one unsplit (1-lane) call, since concurrent lanes overlap
    eng.set_lanes(1)
    eng.segment_device(d_rgb, out)
    tm = eng.last_timing()
    eng.set_lanes(0)
    torch.cuda.synchronize()
    n, k, it = h * w, g.num_clusters, st.no_iters
    bytes_frame = 15 * n + (it + 1) * (16 * n + 40 * k) + it * (16 * n + 48 * k) + 16 * n + 40 * k
    fps = b / (ms / 1e3)
    rec = {"config": name, "image": f"{w}x{h}", "S": g.s, "K": k, "iters": it, "frames": b,
           "lanes": lanes,
           "ms_per_batch": ms, "frames_per_s": fps, "mpix_per_s": fps * n / 1e6,
           "bytes_per_frame": bytes_frame,
           "hbm_frac": bytes_frame * fps / 1e9 / PEAK,
           "stage_ms": {"convert": tm.convert * 1e3,
                        "associate_mean": 1e3 * sum(tm.associate[:-1]) / max(1, len(tm.associate) - 1),
                        "final_associate": tm.associate[-1] * 1e3,
                        "update_mean": 1e3 * sum(tm.update) / max(1, len(tm.update)),
                        "connectivity": tm.connectivity * 1e3}}
    if check:
        import oracle
        t0 = time.time()
        labels, cxy, clab, counts, _ = oracle.segment(host[0], g.s, g.ns_r, g.ns_c,
                                                      st.compactness, no_iters=it)
        ok = (np.array_equal(out[0][0].cpu().numpy(), labels)
              and out[2][0].cpu().numpy().tobytes() == clab.tobytes()
              and out[1][0].cpu().numpy().tobytes() == cxy.tobytes()
              and np.array_equal(out[3][0].cpu().numpy(), counts))
        rec["oracle_bitexact_frame0"] = bool(ok)
        rec["oracle_s"] = round(time.time() - t0, 1)
    del eng, d_rgb, out
    torch.cuda.empty_cache()
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C3,C4,C5")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--md", default=None)
    a = ap.parse_args()
    recs = []
    for name in a.configs.split(","):
        r = run(name, a.reps, a.warmup)
        print(json.dumps(r), flush=True)
        recs.append(r)
    if a.md:
        with open(a.md, "w") as f:
            f.write("# Device throughput per BASELINE config (one B200, tools/bench_configs.py)\n\n")
            f.write("Inputs resident in HBM; CUDA-event timing; bytes per SURVEY §8(d); "
                    f"peak {PEAK} GB/s.  Throughput with the engine's automatic lanes "
                    "(concurrent sub-batches); stage columns from one unsplit call.\n\n")
            f.write("| config | image | S | K | iters | frames/batch | lanes | ms/batch | frames/s | Mpix/s "
                    "| HBM frac | convert | assoc+update pass | final assoc | update | weak | "
                    "frame 0 == oracle |\n|" + "---|" * 17 + "\n")
            for r in recs:
                s = r["stage_ms"]
                f.write(f"| {r['config']} | {r['image']} | {r['S']} | {r['K']} | {r['iters']} | "
                        f"{r['frames']} | {r['lanes']} | {r['ms_per_batch']:.3f} | {r['frames_per_s']:.1f} | "
                        f"{r['mpix_per_s']:.0f} | {r['hbm_frac']:.3f} | {s['convert']:.3f} | "
                        f"{s['associate_mean']:.3f} | {s['final_associate']:.3f} | "
                        f"{s['update_mean']:.3f} | {s['connectivity']:.3f} | "
                        f"{r.get('oracle_bitexact_frame0', 'n/a')} |\n")


if __name__ == "__main__":
    main()

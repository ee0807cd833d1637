"""Device throughput of every BASELINE.json config and PAPER.md Table 1 on one B200.

For each config: synthetic frames from the reference generator
(np.random.default_rng(i).integers(0, 256, (H, W, 3), uint8)), resident in HBM,
W warm-up + R timed batches with CUDA events, per-stage device times, the
SURVEY §8(d) algorithmic bytes per frame and the HBM-roofline fraction.
Frame 0 (seed 0) is checked bit-for-bit against the REFERENCE's own output
hashes (tests/golden/golden_hashes.json, produced by the unmodified reference;
test tooling), or against the C oracle when no hash exists.

Table 1 rows (image sizes at 1000 / 2000 superpixels) are
timed per image twice: one image per call (the paper's setting; the call is
a replayed CUDA graph) and a batch of 16 images per call; gSLICr's published
seconds per image (GTX Titan Black) are printed beside them.

    python tools/bench_configs.py [--configs C1,C2,...|all|table1] [--md out.md]
"""
import argparse
import hashlib
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1509_04232_b200 as spx  # noqa: E402


def measured_peak():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


PEAK, PEAK_SRC = measured_peak()
# name: (W, H, settings kwargs, frames per batch, reference hash key of frame 0)
CONFIGS = {
    "C1": (640, 480, dict(num_superpixels=1200), 256, "frame_C1_640x480"),
    "C2": (1280, 960, dict(num_superpixels=4800), 64, "frame_C2_1280x960"),
    "C3": (1920, 1080, dict(num_superpixels=8000), 128, "large_C3_f0"),
    "C4": (3840, 2160, dict(spixel_size=8, no_iters=10), 8, "large_C4"),
    "C5": (16384, 16384, dict(spixel_size=16), 1, "large_C5"),
}
# gSLICr seconds per image (1000 and 2000 superpixels)
TABLE1 = {(1024, 1024): 0.01, (3631, 3859): 0.12, (963, 1024): 0.01, (1002, 1002): 0.01,
          (933, 800): 0.008}
for (w_, h_), _t in TABLE1.items():
    for k_ in (1000, 2000):
        CONFIGS[f"T1_{w_}x{h_}_k{k_}"] = (w_, h_, dict(num_superpixels=k_), 16,
                                          f"large_T1_{w_}x{h_}_k{k_}")


def golden_hashes():
    with open(os.path.join(REPO, "tests", "golden", "golden_hashes.json")) as fh:
        return json.load(fh)["hashes"]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def frames(h, w, n):
    return np.stack([np.random.default_rng(i).integers(0, 256, (h, w, 3), dtype=np.uint8)
                     for i in range(n)])


def time_calls(eng, d_rgb, out, reps, warm):
    for _ in range(warm):
        eng.segment_device(d_rgb, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        eng.segment_device(d_rgb, out)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def run(name, reps, warm):
    w, h, kw, b, check = CONFIGS[name]
    st = spx.Settings(img_width=w, img_height=h, **kw)
    g = spx.compute_grid(st)
    single_ms = None
    if name.startswith("T1_"):
        # one image per call, as the paper times it (graph replay after 2 calls)
        e1 = spx.SegEngine(st, max_batch=1)
        d1 = torch.from_numpy(frames(h, w, 1)).cuda()
        single_ms = time_calls(e1, d1, e1.allocate_outputs(1), max(reps, 20), max(warm, 3))
        del e1, d1
    eng = spx.SegEngine(st, max_batch=b)
    host = frames(h, w, min(b, 8))
    if b > host.shape[0]:  # repeat the first 8 generator frames (same statistics)
        host = np.concatenate([host] * (b // host.shape[0]) + [host[:b % host.shape[0]]])
    d_rgb = torch.from_numpy(host).cuda()
    out = eng.allocate_outputs(b)
    ms = time_calls(eng, d_rgb, out, reps, warm)
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
           "lanes": lanes, "fused_path": eng.fused_path,
           "ms_per_batch": ms, "frames_per_s": fps, "mpix_per_s": fps * n / 1e6,
           "bytes_per_frame": bytes_frame,
           "hbm_frac": bytes_frame * fps / 1e9 / PEAK,
           "stage_ms": {"convert": tm.convert * 1e3,
                        "associate_mean": 1e3 * sum(tm.associate[:-1]) / max(1, len(tm.associate) - 1),
                        "final_associate": tm.associate[-1] * 1e3,
                        "update_mean": 1e3 * sum(tm.update) / max(1, len(tm.update)),
                        "connectivity": tm.connectivity * 1e3}}
    if single_ms is not None:
        rec["ms_per_image_single_call"] = single_ms
        rec["ms_per_image_batched"] = ms / b
        rec["gslicr_s_per_image"] = TABLE1[(w, h)]
    hashes = golden_hashes()
    got = [out[i][0].cpu().numpy() for i in range(4)]
    if check in hashes:
        m = hashes[check]
        ok = [sha(got[0]), sha(got[1]), sha(got[2]), sha(got[3])] == [
            m["labels"], m["cxy"], m["clab"], m["counts"]]
        rec["frame0_equals_reference"] = bool(ok)
    else:
        import oracle
        labels, cxy, clab, counts, _ = oracle.segment(host[0], g.s, g.ns_r, g.ns_c,
                                                      st.compactness, no_iters=it)
        ok = (np.array_equal(got[0], labels) and got[2].tobytes() == clab.tobytes()
              and got[1].tobytes() == cxy.tobytes() and np.array_equal(got[3], counts))
        rec["frame0_equals_oracle"] = bool(ok)
    del eng, d_rgb, out
    torch.cuda.empty_cache()
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C3,C4,C5", help="names, 'all' or 'table1'")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--md", default=None)
    a = ap.parse_args()
    names = a.configs.split(",")
    if a.configs == "all":
        names = list(CONFIGS)
    elif a.configs == "table1":
        names = [n for n in CONFIGS if n.startswith("T1_")]
    recs = []
    for name in names:
        r = run(name, a.reps, a.warmup)
        print(json.dumps(r), flush=True)
        recs.append(r)
    if a.md:
        with open(a.md, "w") as f:
            f.write("# Device throughput per config (one B200, tools/bench_configs.py)\n\n")
            f.write("Inputs resident in HBM; CUDA-event timing; bytes per SURVEY §8(d); "
                    f"peak {PEAK} GB/s ({PEAK_SRC}).  Throughput with the engine's automatic "
                    "lanes (concurrent sub-batches); stage columns (ms per batch) from one "
                    "unsplit call.  Last column: frame 0 (seed 0) against the reference's own "
                    "output hashes.\n\n")
            f.write("| config | image | S | K | iters | frames/batch | fused | lanes | ms/batch | "
                    "frames/s | Mpix/s | HBM frac | convert | assoc+update pass | final assoc | "
                    "update | weak | frame 0 == reference |\n|" + "---|" * 18 + "\n")
            for r in recs:
                s = r["stage_ms"]
                eq = r.get("frame0_equals_reference", r.get("frame0_equals_oracle", "n/a"))
                f.write(f"| {r['config']} | {r['image']} | {r['S']} | {r['K']} | {r['iters']} | "
                        f"{r['frames']} | {r['fused_path']} | {r['lanes']} | "
                        f"{r['ms_per_batch']:.3f} | {r['frames_per_s']:.1f} | "
                        f"{r['mpix_per_s']:.0f} | {r['hbm_frac']:.3f} | {s['convert']:.3f} | "
                        f"{s['associate_mean']:.3f} | {s['final_associate']:.3f} | "
                        f"{s['update_mean']:.3f} | {s['connectivity']:.3f} | {eq} |\n")
            t1 = [r for r in recs if "gslicr_s_per_image" in r]
            if t1:
                f.write("\n## PAPER.md Table 1 sizes (per image)\n\n")
                f.write("| image | superpixels | S | one image per call (ms) | batched x16 (ms per "
                        "image) | gSLICr (ms, GTX Titan Black) | speed-up (single call) |\n"
                        "|---|---|---|---|---|---|---|\n")
                for r in t1:
                    g_ms = r["gslicr_s_per_image"] * 1e3
                    f.write(f"| {r['image']} | {r['config'].rsplit('_k', 1)[1]} | {r['S']} | "
                            f"{r['ms_per_image_single_call']:.3f} | "
                            f"{r['ms_per_image_batched']:.3f} | {g_ms:.0f} | "
                            f"{g_ms / r['ms_per_image_single_call']:.0f}x |\n")


if __name__ == "__main__":
    main()

"""Randomised parity sweep: engine vs the C oracle on random settings (GPU).

    python tools/fuzz_parity.py [--seconds 300] [--seed 0]

Each case draws an image size, grid interval (spixel_size or num_superpixels),
compactness, iterations, colour space, connectivity, perturbation, tile
length, early-stop threshold and a batch of frames from several generators
(noise, gray, smooth, dark, flat, stripes), runs the batch through
SegEngine.segment_host and compares every frame with oracle.segment bit for
bit.  Prints one line per failing case and a summary; exit status 1 on any
mismatch.
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402  (test infrastructure: the checker)
import paper_1509_04232_b200 as spx  # noqa: E402


def frame(rng, kind, h, w):
    if kind == "noise":
        return rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
    if kind == "gray":
        g = rng.integers(0, 256, (h, w, 1), dtype=np.uint8)
        return np.repeat(g, 3, axis=2)
    if kind == "smooth":
        yy, xx = np.mgrid[0:h, 0:w]
        im = np.stack([xx * 255 // max(w - 1, 1), yy * 255 // max(h - 1, 1),
                       (xx + yy) * 127 // max(w + h - 2, 1)], -1)
        return np.clip(im + rng.integers(-6, 7, (h, w, 3)), 0, 255).astype(np.uint8)
    if kind == "dark":
        return (rng.integers(0, 256, (h, w, 3)) // 40).astype(np.uint8)
    if kind == "flat":
        return np.full((h, w, 3), rng.integers(0, 256, 3), dtype=np.uint8)
    # stripes
    col = rng.integers(0, 256, (7, 3))
    return col[(np.arange(w)[None, :] // max(1, int(rng.integers(1, 9))) +
                np.arange(h)[:, None] // 3) % 7].astype(np.uint8)


# share of cases with large cells (S > 32); SPX_FUZZ_BIG overrides
BIG = float(os.environ.get("SPX_FUZZ_BIG", "0.15"))


def case(rng):
    big = rng.random() < BIG  # large cells (S > 32: strip sums, 16/32 lanes per cell)
    h, w = int(rng.integers(6, 900 if big else 420)), int(rng.integers(6, 900 if big else 560))
    if rng.random() < 0.5:  # half the shapes 128-bit aligned (W % 4 == 0), half anything
        w += (-w) % 4
    kw = {}
    if big:
        kw["spixel_size"] = int(rng.integers(33, 161))
    elif rng.random() < 0.5:
        kw["spixel_size"] = int(rng.integers(2, 41))
    else:
        kw["num_superpixels"] = int(rng.integers(1, max(2, h * w // 16)))
    kw["compactness"] = float(rng.choice([0.5, 1.0, 5.0, 10.0, 20.0, 40.0]))
    kw["no_iters"] = int(rng.integers(1, 9))
    kw["color_space"] = spx.ColorSpace(int(rng.choice([2, 2, 1, 0])))
    c = rng.random()
    if c < 0.15:
        kw["do_enforce_connectivity"] = False
    elif c < 0.35:
        kw["connectivity_mode"] = spx.ConnectivityMode.STRICT
    kw["enable_perturbation"] = bool(rng.random() < 0.3)
    kw["tile_len"] = int(rng.choice([16, 16, 1, 3, 5, 8, 20]))
    if rng.random() < 0.25:
        kw["early_stop_threshold"] = float(rng.choice([0.0, 1.0, 10.0, 100.0]))
    try:
        st = spx.Settings(img_width=w, img_height=h, **kw)
        spx.compute_grid(st)
    except spx.SuperpixError:
        return None
    kinds = ["noise", "gray", "smooth", "dark", "flat", "stripes"]
    b = int(rng.integers(1, 3 if big else 6))
    frames = np.stack([frame(rng, kinds[int(rng.integers(0, len(kinds)))], h, w) for _ in range(b)])
    return st, frames


def check(st, frames):
    g = spx.compute_grid(st)
    eng = spx.SegEngine(st, max_batch=frames.shape[0])
    check.fused += eng.fused_path
    labels, cxy, clab, counts, passes = eng.segment_host(frames)
    conn = 0 if not st.do_enforce_connectivity else (
        2 if st.connectivity_mode is spx.ConnectivityMode.STRICT else 1)
    bad = []
    for i, f in enumerate(frames):
        ol, ox, oc, on, op = oracle.segment(
            f, g.s, g.ns_r, g.ns_c, st.compactness, no_iters=st.no_iters,
            space=st.color_space.value, perturb=st.enable_perturbation, connectivity=conn,
            min_size=st.min_size if st.min_size is not None else None, tile_len=st.tile_len,
            early_stop=st.early_stop_threshold)
        ok = (np.array_equal(labels[i], ol) and cxy[i].tobytes() == ox.tobytes()
              and clab[i].tobytes() == oc.tobytes() and np.array_equal(counts[i], on)
              and int(passes[i]) == int(op))
        if not ok:
            bad.append((i, int((labels[i] != ol).sum())))
    return bad


check.fused = 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=300)
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    t0, n, fails, frames_total = time.time(), 0, 0, 0
    while time.time() - t0 < a.seconds:
        c = case(rng)
        if c is None:
            continue
        st, frames = c
        bad = check(st, frames)
        n += 1
        frames_total += frames.shape[0]
        if bad:
            fails += 1
            print(f"MISMATCH {st} frames {frames.shape} bad {bad}", flush=True)
    print(f"fuzz: {n} cases ({check.fused} on the fused cell path), {frames_total} frames, "
          f"{fails} failing cases ({time.time() - t0:.0f} s)", flush=True)
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()

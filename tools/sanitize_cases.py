"""Small end-to-end cases for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py

Exercises every kernel family once on small inputs and checks each result
against the C oracle (test tooling): the fused cell kernels with and
without accumulation (k_cell), the reduce and the exact fallback
(k_exact_clusters on gray-heavy frames, k_exact_wide for S > 32), strict
connectivity (CCL), lanes inside a captured CUDA graph, early stop (the
pairwise shift tree), row strips, and the generic per-stage kernels
(S < 4).  Exits non-zero on any mismatch.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402  (the checker)
import paper_1509_04232_b200 as spx  # noqa: E402
from paper_1509_04232_b200.strips import segment_strips_local  # noqa: E402


def frames(h, w, seed, kind="noise"):
    rng = np.random.default_rng(seed)
    noise = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
    if kind == "gray":
        g = np.repeat(rng.integers(0, 256, (h, w, 1), dtype=np.uint8), 3, axis=2)
        g[::7] = noise[::7]
        return g
    return noise


def check(name, st, rgb, got):
    g = spx.compute_grid(st)
    conn = 0 if not st.do_enforce_connectivity else (
        2 if st.connectivity_mode is spx.ConnectivityMode.STRICT else 1)
    want = oracle.segment(rgb, g.s, g.ns_r, g.ns_c, st.compactness, no_iters=st.no_iters,
                          connectivity=conn, tile_len=st.tile_len,
                          early_stop=st.early_stop_threshold)
    ok = all(np.asarray(a).tobytes() == np.asarray(b).tobytes() for a, b in zip(got, want[:4]))
    print(f"{name}: {'ok' if ok else 'MISMATCH'}", flush=True)
    return ok


def one(name, st, rgb):
    r = spx.SegEngine(st).perform_segmentation(spx.ImageRGB(rgb))
    return check(name, st, rgb, (r.labels.data, r.spixel_map.centers_xy,
                                 r.spixel_map.centers_lab, r.spixel_map.num_pixels))


def main():
    ok = True
    st = spx.Settings(img_width=160, img_height=120, num_superpixels=75)
    ok &= one("cell path noise", st, frames(120, 160, 1))
    ok &= one("cell path gray (exact fallback)", st, frames(120, 160, 2, "gray"))
    ok &= one("odd frame 99x75 S=9", spx.Settings(img_width=75, img_height=99, spixel_size=9),
              frames(99, 75, 3))
    ok &= one("S=40 (k_exact_wide)", spx.Settings(img_width=200, img_height=180, spixel_size=40,
                                                  no_iters=2), frames(180, 200, 4, "gray"))
    ok &= one("strict", spx.Settings(img_width=96, img_height=64, num_superpixels=24,
                                     connectivity_mode=spx.ConnectivityMode.STRICT),
              frames(64, 96, 5))
    ok &= one("early stop", spx.Settings(img_width=96, img_height=64, num_superpixels=24,
                                         no_iters=8, early_stop_threshold=15.0), frames(64, 96, 6))
    ok &= one("generic S=3", spx.Settings(img_width=40, img_height=30, spixel_size=3, no_iters=2),
              frames(30, 40, 7))
    # lanes in a captured graph: eager, eager, capture, replay
    st = spx.Settings(img_width=96, img_height=64, num_superpixels=24)
    batch = np.stack([frames(64, 96, 10 + i) for i in range(8)])
    eng = spx.SegEngine(st, max_batch=8)
    eng.set_lanes(3)
    d = torch.from_numpy(batch).cuda()
    out = eng.allocate_outputs(8)
    for _ in range(4):
        eng.segment_device(d, out)
    torch.cuda.synchronize()
    for i in (0, 7):
        ok &= check(f"lanes+graph frame {i}", st, batch[i], [t[i].cpu().numpy() for t in out[:4]])
    st = spx.Settings(img_width=160, img_height=200, spixel_size=16, no_iters=3)
    rgb = frames(200, 160, 11)
    ok &= check("3 row strips", st, rgb, segment_strips_local(st, rgb, 3))
    torch.cuda.synchronize()
    print("ALL OK" if ok else "FAILURES", flush=True)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())

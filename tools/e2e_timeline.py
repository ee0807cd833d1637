"""Per-chunk H2D / compute / D2H timeline of the pipelined host path (diagnostic).

Run with SPX_DEBUG_TIMELINE=1 (and optionally CHUNK=N frames per chunk)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1509_04232_b200 as spx  # noqa: E402

B, H, W = 256, 480, 640
st = spx.Settings(img_width=W, img_height=H, num_superpixels=1200)
eng = spx.SegEngine(st, max_batch=B)
K = eng.grid.num_clusters
eng.set_host_chunk(int(os.environ.get("CHUNK", B)))
host = torch.from_numpy(np.random.default_rng(0).integers(0, 256, (B, H, W, 3), dtype=np.uint8)
                        ).pin_memory().numpy()
outs = [[torch.empty(s, dtype=d).pin_memory().numpy() for s, d in
         (((B, H, W), torch.int32), ((B, K, 2), torch.float64), ((B, K, 3), torch.float64),
          ((B, K), torch.int64), ((B,), torch.int32))] for _ in range(2)]
eng.segment_host(host, *outs[0])
steps = int(os.environ.get("STEPS", "4"))
t = time.perf_counter()
for i in range(steps):
    eng.submit_host(host, *outs[i & 1])
eng.wait()
dt = time.perf_counter() - t
print(f"{steps} steps: {dt / steps * 1e3:.2f} ms/step -> {B * steps / dt:.0f} frames/s", flush=True)

"""Small-batch latency of the device API, with and without CUDA graphs (diagnostic).

    python tools/latency.py            # graphs on (default)
    SPX_NO_GRAPHS=1 python tools/latency.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1509_04232_b200 as spx  # noqa: E402

st = spx.Settings(img_width=640, img_height=480, num_superpixels=1200)
for b in (1, 4, 16, 64):
    eng = spx.SegEngine(st, max_batch=b)
    rgb = torch.from_numpy(np.stack([np.random.default_rng(i).integers(0, 256, (480, 640, 3),
                                                                      dtype=np.uint8)
                                     for i in range(b)])).cuda()
    out = eng.allocate_outputs(b)
    for _ in range(5):
        eng.segment_device(rgb, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 50
    e0.record()
    for _ in range(n):
        eng.segment_device(rgb, out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"graphs={'off' if os.environ.get('SPX_NO_GRAPHS') else 'on'} batch {b:3d}: "
          f"{ms * 1e3:8.1f} us per call, {b / ms * 1e3:9.0f} frames/s, "
          f"launches {eng.last_launches()}", flush=True)

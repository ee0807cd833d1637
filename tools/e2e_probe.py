"""Probe host<->device copy rates and the overlapped host path (diagnostic)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1509_04232_b200 as spx

B, H, W = 256, 480, 640
st = spx.Settings(img_width=W, img_height=H, num_superpixels=1200)
eng = spx.SegEngine(st, max_batch=B)
host = np.random.default_rng(0).integers(0, 256, (B, H, W, 3), dtype=np.uint8)
pin = torch.from_numpy(host).pin_memory()
dev = torch.empty_like(pin, device="cuda")
lab_d = torch.empty((B, H, W), dtype=torch.int32, device="cuda")
lab_h = torch.empty((B, H, W), dtype=torch.int32).pin_memory()
for name, fn, nbytes in (("h2d", lambda: dev.copy_(pin, non_blocking=True), pin.numel()),
                         ("d2h", lambda: lab_h.copy_(lab_d, non_blocking=True), lab_h.numel() * 4)):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5): fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 5
    print(f"{name}: {nbytes / dt / 1e9:.1f} GB/s ({dt * 1e3:.2f} ms per {nbytes / 1e6:.0f} MB)")
outs = eng.allocate_outputs(B)
eng.segment_device(dev, outs); torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5): eng.segment_device(dev, outs)
torch.cuda.synchronize()
print(f"device: {(time.perf_counter() - t) / 5 * 1e3:.2f} ms per batch")
K = spx.compute_grid(st).num_clusters
bufs = [torch.empty(s, dtype=d).pin_memory().numpy() for s, d in
        (((B, H, W), torch.int32), ((B, K, 2), torch.float64), ((B, K, 3), torch.float64),
         ((B, K), torch.int64), ((B,), torch.int32))]
ph = pin.numpy()
eng.segment_host(ph, *bufs)
t = time.perf_counter()
for _ in range(5): eng.segment_host(ph, *bufs)
dt = (time.perf_counter() - t) / 5
print(f"host path: {dt * 1e3:.2f} ms per batch -> {B / dt:.0f} frames/s")

import os, sys, time, statistics
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1509_04232_b200 as spx
st = spx.Settings(img_width=640, img_height=480, num_superpixels=1200)
eng = spx.SegEngine(st)
img = spx.ImageRGB(np.random.default_rng(0).integers(0, 256, (480, 640, 3), dtype=np.uint8))
d = torch.from_numpy(img.data.copy()).cuda()[None]; out = eng.allocate_outputs(1)
for _ in range(20): eng.segment_device(d, out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(200): eng.segment_device(d, out)
e1.record(); torch.cuda.synchronize()
print(os.environ.get("SPX_LPC"), "device per frame us", e0.elapsed_time(e1) / 200 * 1e3)
os.environ["SPX_NO_GRAPHS"] = "1"
eng2 = spx.SegEngine(st)
for _ in range(3): eng2.segment_device(d, out)
torch.cuda.synchronize()
tm = eng2.last_timing()
print(" stages us: convert %.1f init %.1f assoc %s update %s conn %.1f total %.1f" % (tm.convert*1e6, tm.init*1e6, [round(a*1e6,1) for a in tm.associate], [round(a*1e6,1) for a in tm.update], tm.connectivity*1e6, tm.total*1e6))
ts = []
for _ in range(300):
    t0 = time.perf_counter(); eng.perform_segmentation(img); ts.append(time.perf_counter() - t0)
print(" perform_segmentation median us", statistics.median(ts) * 1e6)

import os, sys, time, statistics
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1509_04232_b200 as spx
st = spx.Settings(img_width=640, img_height=480, num_superpixels=1200)
eng = spx.SegEngine(st)
img = spx.ImageRGB(np.random.default_rng(0).integers(0, 256, (480, 640, 3), dtype=np.uint8))
k = eng.grid.num_clusters
def pin(shape, dt): return torch.empty(shape, dtype=dt).pin_memory().numpy()
prgb = pin((1,480,640,3), torch.uint8); np.copyto(prgb[0], img.data)
po = (pin((1,480,640), torch.int32), pin((1,k,2), torch.float64), pin((1,k,3), torch.float64), pin((1,k), torch.int64), pin((1,), torch.int32))
def T(name, f, n=300):
    for _ in range(20): f()
    ts=[]
    for _ in range(n):
        t0=time.perf_counter(); f(); ts.append(time.perf_counter()-t0)
    print(f"{name:40s} median {statistics.median(ts)*1e6:8.1f} us  min {min(ts)*1e6:8.1f}")
T("perform_segmentation", lambda: eng.perform_segmentation(img))
T("segment_host pageable", lambda: eng.segment_host(img.data))
T("segment_host pinned in, pageable out", lambda: eng.segment_host(prgb))
T("segment_host pinned in+out", lambda: eng.segment_host(prgb, *po))
T("last_timing", lambda: eng.last_timing())
res = eng.segment_host(img.data)
T("_results", lambda: eng._results(*res, eng.last_timing()))
T("copyto 0.92MB", lambda: np.copyto(prgb[0], img.data))
lab = np.empty((480,640), np.int32)
T("copy 1.23MB labels", lambda: np.copyto(lab, po[0][0]))
T("torch pinned alloc 1.3MB", lambda: torch.empty((1300000,), dtype=torch.uint8, pin_memory=True))
T("LabelMap", lambda: spx.LabelMap(lab))
d = torch.from_numpy(prgb).cuda(); out = eng.allocate_outputs(1)
def dev():
    eng.segment_device(d, out); torch.cuda.synchronize()
T("segment_device + sync", dev)
import ctypes
from paper_1509_04232_b200 import _lib
pin = eng._pinned_input(1)
outs = eng._pinned_outputs(1)
p = lambda a: a.ctypes.data_as(ctypes.c_void_p)
T("_pinned_outputs", lambda: eng._pinned_outputs(1))
T("spx_engine_segment_host block", lambda: eng._lib.spx_engine_segment_host(eng._h, p(pin), 1, *(p(a) for a in outs)))
T("spx_engine_segment_host block fresh", lambda: eng._lib.spx_engine_segment_host(eng._h, p(pin), 1, *(p(a) for a in eng._pinned_outputs(1))))
hb = eng.segment_host(prgb, *po)
T("ctypes segment_host separate pinned", lambda: eng._lib.spx_engine_segment_host(eng._h, p(prgb), 1, *(p(a) for a in po)))
import os
os.environ["SPX_DEBUG_TIMELINE"] = "1"

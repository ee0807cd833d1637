import os, sys
sys.path.insert(0, os.getcwd())
os.environ["SPX_NO_GRAPHS"] = "1"
import numpy as np, torch
import paper_1509_04232_b200 as spx
st = spx.Settings(img_width=640, img_height=480, num_superpixels=1200,
                  connectivity_mode=spx.ConnectivityMode.STRICT)
eng = spx.SegEngine(st, max_batch=256)
eng.set_lanes(1)
d = torch.from_numpy(np.stack([np.random.default_rng(i).integers(0, 256, (480, 640, 3), dtype=np.uint8) for i in range(8)] * 32)).cuda()
out = eng.allocate_outputs(256)
for _ in range(int(os.environ.get("REPS", "2"))): eng.segment_device(d, out)
torch.cuda.synchronize()

"""Probe: does splitting a 256-frame C1 step across concurrent engines/streams
help?  The convert kernel is FP64-pipe bound and the association pass is
issue/MUFU bound, so two half-batches on two streams could overlap one's
convert with the other's association.  Prints device ms per 256 frames for
n_split in (1, 2, 4), and checks the split results equal the single-engine
ones (bitwise).  Needs a GPU.
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1509_04232_b200 as spx  # noqa: E402

W, H, B = 640, 480, 256


def main():
    dev = 0
    torch.cuda.set_device(dev)
    rng = np.random.default_rng(0)
    rgb = torch.from_numpy(rng.integers(0, 256, (B, H, W, 3), dtype=np.uint8)).to(dev)
    st = spx.Settings(img_width=W, img_height=H, num_superpixels=1200, compactness=10,
                      no_iters=5)
    ref = None
    for n in (1, 2, 4, 8):
        b = B // n
        engs = [spx.SegEngine(st, device=dev, max_batch=b) for _ in range(n)]
        outs = [e.allocate_outputs(b) for e in engs]
        streams = [torch.cuda.Stream(dev) for _ in range(n)]
        main_s = torch.cuda.current_stream(dev)

        def step():
            ev = torch.cuda.Event()
            ev.record(main_s)
            for i in range(n):
                streams[i].wait_event(ev)
                engs[i].segment_device(rgb[i * b:(i + 1) * b], outs[i], stream=streams[i])
            for i in range(n):
                e2 = torch.cuda.Event()
                e2.record(streams[i])
                main_s.wait_event(e2)

        for _ in range(3):
            step()
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        steps = 10
        s0.record(main_s)
        for _ in range(steps):
            step()
        s1.record(main_s)
        torch.cuda.synchronize()
        ms = s0.elapsed_time(s1) / steps
        labels = torch.cat([o[0] if isinstance(o, (tuple, list)) else o.labels for o in outs])
        if ref is None:
            ref = labels.clone()
        same = bool(torch.equal(labels, ref))
        print(f"split={n}: {ms:.3f} ms/256 frames  {B / ms * 1e3:.0f} frames/s  equal={same}",
              flush=True)


if __name__ == "__main__":
    main()

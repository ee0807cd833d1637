"""Diagnostic probes of the engine on a B200 (development; not part of the product).

    python tools/probe.py latency          # device API, 1..64 frames per call
    python tools/probe.py pseg [--n 300]   # SegEngine.perform_segmentation per frame
    python tools/probe.py lanes [--configs C1,C2,C3,C4] [--lanes 1,2,3,4]
    python tools/probe.py copies           # PCIe rates, device step, host pipeline
    SPX_DEBUG_TIMELINE=1 python tools/probe.py timeline [--chunk N] [--steps K]

latency  -- device-resident segment_device calls of 1, 4, 16, 64 VGA frames
            (CUDA-graph replays after two eager calls); SPX_NO_GRAPHS=1 turns
            graphs off for comparison.
pseg     -- the drop-in per-frame call (host numpy in, SegResult out): median
            wall time, and the pieces it is made of (pinned staging copy,
            native host call, timing read, result objects).
lanes    -- device ms per batch for each lane count (concurrent sub-batches,
            engine.cu) and the automatic choice, on the BASELINE configs.
copies   -- H2D / D2H copy rates of one 256-frame VGA step, the device step,
            and the pipelined host path (spx_engine_segment_host).
timeline -- per-chunk H2D / compute / D2H event timeline of submit_host
            (printed by the native engine when SPX_DEBUG_TIMELINE is set).
"""
import argparse
import ctypes
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1509_04232_b200 as spx  # noqa: E402

VGA = dict(img_width=640, img_height=480, num_superpixels=1200)


def frames(n, h=480, w=640):
    return np.stack([np.random.default_rng(i).integers(0, 256, (h, w, 3), dtype=np.uint8)
                     for i in range(n)])


def timed(fn, n, warm=20):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


def device_ms(eng, rgb, out, reps):
    for _ in range(5):
        eng.segment_device(rgb, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        eng.segment_device(rgb, out)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def latency(a):
    st = spx.Settings(**VGA)
    graphs = "off" if os.environ.get("SPX_NO_GRAPHS") else "on"
    for b in (1, 4, 16, 64):
        eng = spx.SegEngine(st, max_batch=b)
        rgb = torch.from_numpy(frames(b)).cuda()
        ms = device_ms(eng, rgb, eng.allocate_outputs(b), 50)
        print(f"graphs={graphs} batch {b:3d}: {ms * 1e3:8.1f} us per call, "
              f"{b / ms * 1e3:9.0f} frames/s, launches {eng.last_launches()}", flush=True)


def pseg(a):
    st = spx.Settings(**VGA)
    eng = spx.SegEngine(st)
    img = spx.ImageRGB(frames(1)[0])
    med = timed(lambda: eng.perform_segmentation(img), a.n)
    print(f"perform_segmentation 640x480: median {med * 1e6:.1f} us "
          f"(device {eng.last_timing().total * 1e6:.1f} us)")
    pin = eng._pinned_input(1)
    outs = eng._pinned_outputs(1)
    p = lambda x: x.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    parts = {
        "pinned staging copy (0.92 MB)": lambda: np.copyto(pin[0], img.data),
        "fresh pinned result block": lambda: eng._pinned_outputs(1),
        "native host call (H2D, graph, one D2H)": lambda: eng._lib.spx_engine_segment_host(
            eng._h, p(pin), 1, *(p(x) for x in outs)),
        "stage timing read": eng.last_timing,
        "result objects": lambda: spx.SegResult(
            spx.LabelMap._trusted(outs[0][0]),
            spx.SuperpixelMap(eng.grid, outs[1][0], outs[2][0], outs[3][0]),
            eng.last_timing()),
    }
    for name, fn in parts.items():
        print(f"  {name:42s} {timed(fn, a.n) * 1e6:8.1f} us")
    d = torch.from_numpy(frames(1)).cuda()
    out = eng.allocate_outputs(1)

    def dev():
        eng.segment_device(d, out)
        torch.cuda.synchronize()
    print(f"  {'segment_device + synchronize':42s} {timed(dev, a.n) * 1e6:8.1f} us")


LANE_CONFIGS = {
    "C1": (640, 480, dict(num_superpixels=1200), 256),
    "C2": (1280, 960, dict(num_superpixels=4800), 64),
    "C3": (1920, 1080, dict(num_superpixels=8000), 128),
    "C4": (3840, 2160, dict(spixel_size=8, no_iters=10), 8),
}


def lanes(a):
    for name in a.configs.split(","):
        w, h, kw, b = LANE_CONFIGS[name]
        rgb = torch.from_numpy(
            np.random.default_rng(0).integers(0, 256, (b, h, w, 3), dtype=np.uint8)).cuda()
        eng = spx.SegEngine(spx.Settings(img_width=w, img_height=h, **kw), max_batch=b)
        outs = eng.allocate_outputs(b)
        for n in [int(x) for x in a.lanes.split(",")] + [0]:
            eng.set_lanes(n)
            ms = device_ms(eng, rgb, outs, 8)
            tag = f"auto({eng.last_lanes()})" if n == 0 else str(n)
            print(f"{name} lanes={tag}: {ms:.3f} ms/batch of {b}  {b / ms * 1e3:.1f} frames/s",
                  flush=True)
        del eng, outs, rgb
        torch.cuda.empty_cache()


def _pinned_set(b, k, h=480, w=640):
    return [torch.empty(s, dtype=d).pin_memory().numpy() for s, d in
            (((b, h, w), torch.int32), ((b, k, 2), torch.float64), ((b, k, 3), torch.float64),
             ((b, k), torch.int64), ((b,), torch.int32))]


def copies(a):
    b = 256
    st = spx.Settings(**VGA)
    eng = spx.SegEngine(st, max_batch=b)
    pin = torch.from_numpy(frames(8).repeat(32, axis=0)).pin_memory()
    dev = torch.empty_like(pin, device="cuda")
    lab_d = torch.empty((b, 480, 640), dtype=torch.int32, device="cuda")
    lab_h = torch.empty((b, 480, 640), dtype=torch.int32).pin_memory()
    for name, fn, nbytes in (("h2d", lambda: dev.copy_(pin, non_blocking=True), pin.numel()),
                             ("d2h", lambda: lab_h.copy_(lab_d, non_blocking=True),
                              lab_h.numel() * 4)):
        def sync_fn(f=fn):
            f()
            torch.cuda.synchronize()
        dt = timed(sync_fn, 5, warm=1)
        print(f"{name}: {nbytes / dt / 1e9:.1f} GB/s ({dt * 1e3:.2f} ms per {nbytes / 1e6:.0f} MB)")
    print(f"device: {device_ms(eng, dev, eng.allocate_outputs(b), 5):.2f} ms per batch")
    bufs = _pinned_set(b, eng.grid.num_clusters)
    dt = timed(lambda: eng.segment_host(pin.numpy(), *bufs), 5, warm=1)
    print(f"host path: {dt * 1e3:.2f} ms per batch -> {b / dt:.0f} frames/s")


def timeline(a):
    b = 256
    eng = spx.SegEngine(spx.Settings(**VGA), max_batch=b)
    eng.set_host_chunk(a.chunk or b)
    host = torch.from_numpy(frames(8).repeat(32, axis=0)).pin_memory().numpy()
    outs = [_pinned_set(b, eng.grid.num_clusters) for _ in range(2)]
    eng.segment_host(host, *outs[0])
    t = time.perf_counter()
    for i in range(a.steps):
        eng.submit_host(host, *outs[i & 1])
    eng.wait()
    dt = time.perf_counter() - t
    print(f"{a.steps} steps: {dt / a.steps * 1e3:.2f} ms/step -> {b * a.steps / dt:.0f} frames/s")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("probe", choices=["latency", "pseg", "lanes", "copies", "timeline"])
    ap.add_argument("--n", type=int, default=300)
    ap.add_argument("--configs", default="C1,C2,C3,C4")
    ap.add_argument("--lanes", default="1,2,3,4,8")
    ap.add_argument("--chunk", type=int, default=0)
    ap.add_argument("--steps", type=int, default=4)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    globals()[a.probe](a)


if __name__ == "__main__":
    main()

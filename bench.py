"""Throughput benchmark: full 5-iteration SLIC at 640x480, K=1200 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl ours|reference]

--gpus N > 1 outside torchrun re-executes itself as N ranks under
torch.distributed.run (127.0.0.1); under torchrun WORLD_SIZE must equal N.

One "step" segments a batch of B synthetic 640x480 frames (the reference's
generator: np.random.default_rng(i).integers(0, 256, (480, 640, 3), uint8))
through the whole pipeline -- convert, init, association x6, update x5, weak
connectivity x2 -- with m=10, LAB, tile_len 16 (S=16, 30x40 clusters).
Frames are sharded across ranks with no collective (weak scaling: B frames
per GPU per step).  Time is measured with CUDA events on the launching
stream, bracketed by barrier + synchronize, max over ranks.

The JSON line carries: value (frames/s, whole job, inputs resident in HBM),
e2e (same metric through the C ABI host-buffer call, H2D + D2H inside the
timed region), roofline (association kernel: algorithmic bytes / measured
pass time vs MEASURED_PEAKS.json), cpu_baseline (the reference itself on the
host cores, rank 0 at N=1), clocks sampled during the timed region.

--impl reference runs the unmodified reference (oracle/_ref, its SegEngine
with the thread-pool backend on all host cores) on the same workload.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

W, H, K_SPX, ITERS, M = 640, 480, 1200, 5, 10.0
METRIC = "frames/s and Mpix/s at 640x480 K~1200 5 iters (1/2/4/8 B200); %HBM roofline"


def synthetic_frames(first, count):
    return np.stack([np.random.default_rng(first + i).integers(0, 256, (H, W, 3), dtype=np.uint8)
                     for i in range(count)])


def algorithmic_bytes(n_px, k, iters):
    """B = 15N + (I+1)(16N+40K) + I(16N+48K) + 16N + 40K per frame."""
    return 15 * n_px + (iters + 1) * (16 * n_px + 40 * k) + iters * (16 * n_px + 48 * k) + 16 * n_px + 40 * k


def measured_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks / clock-event reasons sampled during the timed region.

    NVML every 5 ms (nvidia-smi every 0.2 s if NVML is unavailable).
    """

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    BITS = [0x8, 0x40, 0x20, 0x4]  # nvmlClocksEventReason* / ThrottleReason*

    def __init__(self, dev):
        self.dev = dev
        self.samples = []  # (sm_mhz, max_mhz, set of reason names)
        self._stop = threading.Event()
        self._t = None

    def _nvml_handle(self):
        import pynvml
        import torch
        pynvml.nvmlInit()
        try:
            props = torch.cuda.get_device_properties(self.dev)
            bus = f"{props.pci_domain_id:08x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            idx = int(str(self.dev).split(":")[-1]) if ":" in str(self.dev) else int(self.dev)
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(idx)

    def _init(self):
        """NVML setup, done before the timed region starts (it can take longer
        than a short timed region)."""
        self._nv = None
        try:
            nv, h = self._nvml_handle()
            self._get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons",
                                        getattr(nv, "nvmlDeviceGetCurrentClocksThrottleReasons",
                                                None))
            self._max = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self._nv, self._h = nv, h
        except Exception:
            pass

    def _sample(self):
        if self._nv is not None:
            try:
                nv, h = self._nv, self._h
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                bits = self._get_reasons(h) if self._get_reasons else 0
                self.samples.append((float(sm), self._max,
                                     {n for n, b in zip(self.NAMES, self.BITS) if bits & b}))
            except Exception:
                pass
            return
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        idx = str(self.dev).split(":")[-1]
        try:
            out = subprocess.run(["nvidia-smi", "-i", idx, f"--query-gpu={q}",
                                  "--format=csv,noheader,nounits"], capture_output=True,
                                 text=True, timeout=5).stdout.strip()
            v = [x.strip() for x in out.split(",")]
            if len(v) >= 6 and v[0].replace(".", "").isdigit():
                self.samples.append((float(v[0]), float(v[1]),
                                     {n for n, x in zip(self.NAMES, v[2:6]) if x.lower() == "active"}))
        except Exception:
            pass

    def _run(self):
        period = 0.005 if self._nv is not None else 0.2
        while not self._stop.wait(period):
            self._sample()

    def __enter__(self):
        self._init()
        self._sample()  # one sample as the timed region opens
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": sorted(set().union(*(s[2] for s in self.samples))),
                "samples": len(self.samples)}


def reference_package():
    import oracle
    return oracle.reference_package()


def cpu_reference_rate(seconds, max_frames):
    """Reference SegEngine (thread pool, all host cores) on C1 frames; frames/s."""
    sp = reference_package()
    if sp is None:
        return None
    cores = os.cpu_count() or 1
    st = sp.Settings(img_width=W, img_height=H, num_superpixels=K_SPX, compactness=M,
                     no_iters=ITERS)
    eng = sp.SegEngine(st, backend="par", workers=cores)
    eng.perform_segmentation(sp.ImageRGB(synthetic_frames(0, 1)[0]))  # warm-up (cli.py:171-178)
    n = 0
    t0 = time.perf_counter()
    busy = 0.0
    while n < max_frames and (time.perf_counter() - t0) < seconds:
        img = sp.ImageRGB(synthetic_frames(n, 1)[0])
        busy += eng.perform_segmentation(img).timing.total
        n += 1
    return {"value": n / busy, "unit": "frames/s", "cores": cores, "kind": "reference",
            "sample": f"{n} synthetic 640x480 frames (seeds 0..{n - 1}), reference SegEngine "
                      f"backend=par workers={cores}, sum of timing.total (cli.py _timed_runs method)"}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def free_port():
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def relaunch_ranks(n):
    """`python bench.py --gpus N` outside torchrun: re-exec this command as N
    ranks (one process per GPU) under torch.distributed.run on 127.0.0.1.
    Rank 0 prints the JSON line; the exit code is the launcher's."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def bench_config(B, world):
    """The workload both arms report (identical dicts: the driver compares them)."""
    return {"workload": "C1: 640x480 RGB, K=1200 (S=16, 30x40 grid), m=10, 5 iters, LAB, "
                        "weak connectivity",
            "frames_per_gpu_per_step": B, "global_batch": B * world,
            "parallelism": f"frame-sharded x{world} (no collective)",
            "l2": f"inputs > L2: {B * H * W * 3 / 1e6:.0f} MB RGB + {B * H * W * 12 / 1e6:.0f} MB "
                  f"Lab per GPU per step"}


def run_reference(args):
    world, rank, _ = dist_setup()
    if rank != 0:
        return 0
    sp = reference_package()
    if sp is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return 0
    cores = os.cpu_count() or 1
    st = sp.Settings(img_width=W, img_height=H, num_superpixels=K_SPX, compactness=M,
                     no_iters=ITERS)
    eng = sp.SegEngine(st, backend="par", workers=cores)
    per_step = args.ref_frames
    frames = [sp.ImageRGB(f) for f in synthetic_frames(0, per_step)]
    for _ in range(args.warmup):
        eng.perform_segmentation(frames[0])
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        for f in frames:
            eng.perform_segmentation(f)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = per_step * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(args.batch, world),
        "mpix_per_s": value * W * H / 1e6,
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": cores, "kind": "reference",
                         "sample": f"bounded sample of the workload: {per_step} frames (seeds "
                                   f"0..{per_step - 1}) per step x {args.steps} steps, reference "
                                   f"SegEngine backend=par workers={cores} (oracle/_ref: the "
                                   f"unmodified reference compiled here)"},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1509_04232_b200 as spx

    world, rank, local = dist_setup()
    # SPX_BENCH_BACKEND=gloo: functional check of the multi-rank path on fewer
    # GPUs than ranks (ranks share devices; never a timing configuration)
    backend = os.environ.get("SPX_BENCH_BACKEND", "nccl")
    if world > 1:
        torch.cuda.set_device(local % torch.cuda.device_count())
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    red_dev = dev if backend == "nccl" else "cpu"  # where the max-over-ranks scalars live
    B = args.batch
    st = spx.Settings(img_width=W, img_height=H, num_superpixels=K_SPX, compactness=M,
                      no_iters=ITERS)
    grid = spx.compute_grid(st)
    K = grid.num_clusters
    eng = spx.SegEngine(st, device=dev, max_batch=B)
    # Shard: rank r owns frames [r*B, (r+1)*B) of the global batch (no collective).
    host = synthetic_frames(rank * B, B)
    rgb = torch.from_numpy(host).to(dev)
    outs = eng.allocate_outputs(B)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(max(args.warmup, 3)):
        eng.segment_device(rgb, outs)
    torch.cuda.synchronize()

    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    assoc_ms, update_ms = [], []
    launches = 0
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        start.record(stream)
        for _ in range(args.steps):
            eng.segment_device(rgb, outs)
            launches += eng.last_launches()
        end.record(stream)
        clk._sample()  # the queued steps are still running
        torch.cuda.synchronize()
    barrier()
    ms = start.elapsed_time(end)
    lanes = eng.last_lanes()
    # Per-kernel stage times: the timed steps run `lanes` concurrent sub-batches
    # whose kernels overlap, so the roofline's kernel durations come from one
    # more step of the same 256 frames run unsplit (one lane) right after the
    # timed region (device events around each stage launch).
    eng.set_lanes(1)
    eng.segment_device(rgb, outs)
    tm = eng.last_timing()
    eng.set_lanes(0)
    torch.cuda.synchronize()
    assoc_ms = [t * 1e3 for t in tm.associate]
    update_ms = [t * 1e3 for t in tm.update]
    if world > 1:
        t = torch.tensor([ms], device=red_dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    frames_total = B * world * args.steps
    value = frames_total / (ms / 1e3)

    # ---- end to end through the C ABI host-buffer call (pinned buffers) ----
    # Steps are submitted back to back (SegEngine.submit_host: one H2D / compute /
    # D2H pipeline across batches, as a video stream would use it); every
    # step's input upload and result download is inside the timed region.
    pin_rgb = torch.from_numpy(host).pin_memory().numpy()
    outs = [[torch.empty(shape, dtype=dt).pin_memory().numpy() for shape, dt in
             (((B, H, W), torch.int32), ((B, K, 2), torch.float64), ((B, K, 3), torch.float64),
              ((B, K), torch.int64), ((B,), torch.int32))] for _ in range(2)]
    e2e_steps = args.steps
    # one chunk per step (steps overlap each other's copies; 128-frame chunks measure
    # the same, 64 and 32 lower); SPX_E2E_CHUNK overrides for experiments
    eng.set_host_chunk(int(os.environ.get("SPX_E2E_CHUNK", B)))
    eng.segment_host(pin_rgb, *outs[0])  # warm staging
    barrier()
    t0 = time.perf_counter()
    for i in range(e2e_steps):
        eng.submit_host(pin_rgb, *outs[i & 1])
    eng.wait()
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], device=red_dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = B * world * e2e_steps / e2e_s
    h2d = B * H * W * 3
    d2h = B * (H * W * 4 + K * (16 + 24 + 8) + 4)

    if rank == 0:
        peak, peak_kind = measured_peaks()
        n_px = B * H * W
        # Dominant kernel: the fused association + centre-update pass k_cell<ACC>
        # (ITERS launches per step).  Algorithmic bytes per SURVEY.md §8(d):
        # association 16 B/px + 40 B/cluster, update 16 B/px + 48 B/cluster.
        acc_ms = assoc_ms[:ITERS] if len(assoc_ms) > ITERS else assoc_ms
        acc_mean = statistics.mean(acc_ms)
        acc_bytes = (16 + 16) * n_px + (40 + 48) * K * B
        achieved = acc_bytes / (acc_mean / 1e3) / 1e9
        final_ms = assoc_ms[-1]
        final_bytes = 16 * n_px + 40 * K * B
        traffic = None
        prof = os.path.join(REPO, "profiles", "ncu_assoc_traffic.json")
        if os.path.exists(prof):
            try:
                with open(prof) as fh:
                    pt = json.load(fh)
                traffic = pt["dram_bytes_per_pixel"] * n_px
            except Exception:
                traffic = None
        frame_bytes = algorithmic_bytes(H * W, K, ITERS)
        cpu = None
        if world == 1 and not args.no_cpu:
            cpu = cpu_reference_rate(args.cpu_seconds, args.cpu_frames)
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "dtype_note": "results binary64-identical to the reference; distances filtered in "
                          "fp32 under a certified error bound (uncertain pixels redone in "
                          "binary64), Lab conversion and all sums in binary64",
            "data": "synthetic",
            "config": bench_config(B, world),
            "engine": {"lanes": lanes, "backend": backend if world > 1 else None},
            "mpix_per_s": value * H * W / 1e6,
            "frame_roofline": {"bytes_per_frame": frame_bytes,
                               "achieved_gbs": value / world * frame_bytes / 1e9,
                               "frac": value / world * frame_bytes / 1e9 / peak},
            "roofline": {"kernel": "k_cell<ACC>: fused association + centre-update pass",
                         "bound": "hbm", "achieved": achieved, "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "bytes_per_launch": acc_bytes,
                         "bytes_note": "algorithmic = (16+16) B/px + (40+48) B/cluster per "
                                       "SURVEY §8(d); fused compulsory traffic is 12 B/px "
                                       "read + 4 B/px write + cluster sums",
                         "limiter": "issue slots / MUFU (18 square roots per pixel), not HBM: "
                                    "DESIGN.md section 4",
                         "mean_pass_ms": acc_mean,
                         "stage_source": "one unsplit (1-lane) step after the timed region",
                         "final_assoc": {"ms": final_ms, "bytes": final_bytes,
                                         "frac": final_bytes / (final_ms / 1e3) / 1e9 / peak},
                         "convert": {"ms": tm.convert * 1e3, "bytes": 15 * n_px,
                                     "frac": 15 * n_px / tm.convert / 1e9 / peak},
                         "stage_ms": {"convert": tm.convert * 1e3, "init": tm.init * 1e3,
                                      "associate": assoc_ms, "update": update_ms,
                                      "connectivity": tm.connectivity * 1e3,
                                      "total": tm.total * 1e3}},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "frames/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": e2e_steps,
                    "path": "spx_engine_submit_host x steps + spx_engine_wait (C ABI, pinned host buffers, pipelined across steps)"},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


C5_N, C5_S = 16384, 16
METRIC_C5 = "images/s and Mpix/s, 16384x16384 S=16 5 iters, row strips (1/2/4/8 B200)"


def c5_settings():
    import paper_1509_04232_b200 as spx
    return spx.Settings(img_width=C5_N, img_height=C5_N, spixel_size=C5_S, no_iters=ITERS)


def c5_image():
    return np.random.default_rng(0).integers(0, 256, (C5_N, C5_N, 3), dtype=np.uint8)


def c5_config(world):
    return {"workload": "C5: 16384x16384 RGB (268 Mpx), S=16 (1024x1024 grid, 1,048,576 "
                        "clusters), m=10, 5 iters, LAB, weak connectivity",
            "parallelism": f"row strips x{world}: halo centres, boundary-cluster partial sums "
                           f"and S label rows exchanged with the vertical neighbours per "
                           f"iteration (NCCL send/recv over NVLink)",
            "global_batch": 1, "l2": "inputs > L2: 805 MB RGB + 3.2 GB Lab per image"}


def run_reference_c5(args):
    """Reference arm for C5: the reference SegEngine (all host cores) on a
    bounded band of the image per step, scaled to images/s."""
    world, rank, _ = dist_setup()
    if rank != 0:
        return 0
    sp = reference_package()
    if sp is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return 0
    cores = os.cpu_count() or 1
    rows = args.ref_rows
    band = c5_image()[:rows]
    st = sp.Settings(img_width=C5_N, img_height=rows, spixel_size=C5_S, no_iters=ITERS)
    eng = sp.SegEngine(st, backend="par", workers=cores)
    img = sp.ImageRGB(band)
    for _ in range(args.warmup):
        eng.perform_segmentation(img)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        eng.perform_segmentation(img)
        times.append(time.perf_counter() - t0)
    per_image = statistics.mean(times) * C5_N / rows
    value = 1.0 / per_image
    print(json.dumps({
        "impl": "reference", "metric": METRIC_C5, "value": value, "unit": "images/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * per_image, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": c5_config(world),
        "mpix_per_s": value * C5_N * C5_N / 1e6,
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": cores, "kind": "reference",
                         "sample": f"bounded sample: a {C5_N}x{rows} band of the image per step "
                                   f"(x{args.steps}), reference SegEngine backend=par "
                                   f"workers={cores}, scaled by {C5_N}/{rows}"},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0}}))
    return 0


def run_ours_c5(args):
    """C5: one 16384^2 image per step, row strips over the ranks (strong scaling)."""
    import torch
    import torch.distributed as dist

    from paper_1509_04232_b200.sharding import strip_plan
    from paper_1509_04232_b200.strips import DistComm, LocalComm, StripEngine, _run, strip_window

    world, rank, local = dist_setup()
    backend = os.environ.get("SPX_BENCH_BACKEND", "nccl")
    dev = local % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    st = c5_settings()
    import paper_1509_04232_b200 as spx
    g = spx.compute_grid(st)
    plan = strip_plan(C5_N, g.s, g.ns_r, world)[rank]
    y0, y1 = strip_window(st, rank, world)
    host = c5_image()
    window_host = torch.from_numpy(np.ascontiguousarray(host[y0:y1])).pin_memory()
    del host
    window = window_host.to(dev)
    strip = StripEngine(st, plan.cell_row_lo, plan.cell_row_hi, dev)
    comm = DistComm(rank, world, strip) if world > 1 else LocalComm([strip])
    stream = torch.cuda.current_stream(dev)

    def step(win):
        strip.begin(win)
        _run([strip], comm)
        return strip.finish()

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(max(args.warmup, 3)):
        step(window)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step(window)
        e1.record(stream)
        clk._sample()
        torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1)
    red_dev = dev if backend == "nccl" else "cpu"
    if world > 1:
        t = torch.tensor([ms], device=red_dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = args.steps / (ms / 1e3)
    # end to end: the rank's RGB window uploaded from pinned host memory and
    # its own rows / clusters' results read back, every step
    n_own = strip.own_clusters
    outs_host = [torch.empty((plan.y_hi - plan.y_lo, C5_N), dtype=torch.int32).pin_memory(),
                 torch.empty((n_own, 2), dtype=torch.float64).pin_memory(),
                 torch.empty((n_own, 3), dtype=torch.float64).pin_memory(),
                 torch.empty((n_own,), dtype=torch.int64).pin_memory()]
    barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        window.copy_(window_host, non_blocking=True)
        res = step(window)
        for hb, d in zip(outs_host, res):
            hb.copy_(d, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([e2e_ms], device=red_dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    h2d = window_host.numel() * world
    d2h = sum(t.numel() * t.element_size() for t in outs_host) * world
    if rank == 0:
        peak, peak_kind = measured_peaks()
        n_px = C5_N * C5_N
        frame_bytes = algorithmic_bytes(n_px, g.num_clusters, ITERS)
        cpu = None
        if world == 1 and not args.no_cpu:
            sp = reference_package()
            if sp is not None:
                rows = args.ref_rows
                band = np.random.default_rng(0).integers(0, 256, (C5_N, C5_N, 3),
                                                         dtype=np.uint8)[:rows]
                cores = os.cpu_count() or 1
                rst = sp.Settings(img_width=C5_N, img_height=rows, spixel_size=C5_S,
                                  no_iters=ITERS)
                reng = sp.SegEngine(rst, backend="par", workers=cores)
                t0 = time.perf_counter()
                reng.perform_segmentation(sp.ImageRGB(band))
                per_image = (time.perf_counter() - t0) * C5_N / rows
                cpu = {"value": 1.0 / per_image, "unit": "images/s", "cores": cores,
                       "kind": "reference",
                       "sample": f"a {C5_N}x{rows} band, reference SegEngine par x{cores}, "
                                 f"scaled by {C5_N}/{rows}"}
        line = {
            "metric": METRIC_C5, "value": value, "unit": "images/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": c5_config(world),
            "mpix_per_s": value * n_px / 1e6,
            "frame_roofline": {"bytes_per_image": frame_bytes,
                               "achieved_gbs": value * frame_bytes / 1e9 / world,
                               "frac": value * frame_bytes / 1e9 / world / peak,
                               "peak": peak, "peak_kind": peak_kind,
                               "note": "SURVEY §8(d) bytes of the whole image / time, per GPU"},
            "cpu_baseline": cpu,
            "e2e": {"value": args.steps / (e2e_ms / 1e3), "unit": "images/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "path": "per rank: RGB window H2D (pinned), strip engine, own results D2H"},
            "gpu_launches": None, "clocks": clk.summary(),
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=256, help="frames per GPU per step")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-frames", type=int, default=8, help="reference arm: frames per step")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--cpu-frames", type=int, default=400)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--workload", default="c1", choices=["c1", "c5"],
                    help="c1: the BASELINE headline (default); c5: 16384^2 row strips")
    ap.add_argument("--ref-rows", type=int, default=1024,
                    help="c5 reference arm / cpu_baseline: rows of the bounded band")
    args = ap.parse_args()
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_ranks(args.gpus)
    world = dist_setup()[0]
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    if args.workload == "c5":
        return run_reference_c5(args) if args.impl == "reference" else run_ours_c5(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

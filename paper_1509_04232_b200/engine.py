"""GPU segmentation engine with the reference's SegEngine API.

superpix/engine.py runs the stage sequence of engine.py:125-230 from Python,
calling one CPU kernel per band.  Here the whole sequence -- convert, init,
optional perturbation, association x(iters+1), update x iters, connectivity
-- is one call into the native engine (libspx.so, csrc/engine.cu), which
owns HBM-resident buffers sized at construction and launches each stage once
over a whole batch of frames.  The Python layer validates, moves frames in
and results out, and builds the same SegResult / StageTiming objects.

Backends: "cuda" is the native engine.  The reference's "seq" and "par"
names are accepted as aliases of it (a drop-in caller keeps working and gets
identical labels, which the reference guarantees across its own backends);
`workers` is validated as the reference does and otherwise ignored.
"""

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib, kernels, slic_core
from .connectivity import default_min_size
from .errors import DimensionMismatchError, InvalidSettingsError
from .slic_core import ConnectivityMode, LabelMap, SuperpixelMap

BACKENDS = ("cuda", "seq", "par")


def band_bounds(n, workers):
    """Split [0, n) into `workers` contiguous half-open ranges (engine.py:23-25)."""
    return [((i * n) // workers, ((i + 1) * n) // workers) for i in range(workers)]


@dataclass(frozen=True)
class StageTiming:
    """Seconds per stage (device time).  associate/update: one entry per pass."""

    convert: float
    init: float
    perturb: float
    associate: tuple
    update: tuple
    connectivity: float
    total: float


@dataclass(frozen=True)
class SegResult:
    labels: LabelMap
    spixel_map: SuperpixelMap
    timing: StageTiming


def _native_settings(settings, grid):
    conn = 0
    if settings.do_enforce_connectivity:
        conn = 1 if settings.connectivity_mode is ConnectivityMode.WEAK else 2
    min_size = settings.min_size if settings.min_size is not None else default_min_size(grid.s)
    st = _lib.SpxSettings()
    st.width, st.height = settings.img_width, settings.img_height
    st.s, st.ns_r, st.ns_c = grid.s, grid.ns_r, grid.ns_c
    st.compactness = float(settings.compactness)
    st.no_iters = int(settings.no_iters)
    st.color_space = int(settings.color_space.value)
    st.connectivity = conn
    st.perturb = int(bool(settings.enable_perturbation))
    st.tile_len = int(settings.tile_len)
    st.min_size = int(min_size)
    st.early_stop = -1.0 if settings.early_stop_threshold is None else float(settings.early_stop_threshold)
    return st


class SegEngine:
    """Reusable pipeline for frames of one size (engine.py:86-119 API).

    Buffers for up to `max_batch` frames live on `device` for the engine's
    lifetime.  One engine runs one call at a time; use one engine per thread.
    """

    def __init__(self, settings, backend="cuda", workers=None, kernel_impl="auto",
                 device=None, max_batch=1):
        self.settings = settings
        self.grid = slic_core.compute_grid(settings)
        self.kernel = kernels.get_impl(kernel_impl)
        if backend not in BACKENDS:
            raise InvalidSettingsError(f"unknown backend {backend!r}")
        if backend == "par" and workers is not None and workers < 1:
            raise InvalidSettingsError(f"workers must be >= 1, got {workers}")
        self.backend_name = backend
        self._workers = 1 if workers is None else int(workers)
        import torch  # device plumbing only
        self._torch = torch
        if device is None:
            device = torch.cuda.current_device() if torch.cuda.is_available() else 0
        self.device = int(device)
        self.max_batch = int(max_batch)
        self._pending = []  # host arrays of submitted batches, kept alive until wait()
        lib = _lib.load()
        self._st = _native_settings(settings, self.grid)
        handle = ctypes.c_void_p()
        _lib.check(lib.spx_engine_create(ctypes.byref(self._st), self.max_batch, self.device,
                                         ctypes.byref(handle)), "SegEngine")
        self._h = handle
        self._lib = lib

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                self._lib.spx_engine_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def workers(self):
        return self._workers

    @property
    def num_clusters(self):
        return self.grid.num_clusters

    # ---- device-resident batch API -------------------------------------------------

    def allocate_outputs(self, batch):
        """Device tensors for `batch` frames of results (labels, cxy, clab, counts, passes)."""
        t = self._torch
        dev = t.device("cuda", self.device)
        st = self.settings
        k = self.grid.num_clusters
        return (t.empty((batch, st.img_height, st.img_width), dtype=t.int32, device=dev),
                t.empty((batch, k, 2), dtype=t.float64, device=dev),
                t.empty((batch, k, 3), dtype=t.float64, device=dev),
                t.empty((batch, k), dtype=t.int64, device=dev),
                t.empty((batch,), dtype=t.int32, device=dev))

    def segment_device(self, rgb, out=None, stream=None):
        """Segment a CUDA uint8 tensor (B, H, W, 3); asynchronous on `stream`.

        Returns (labels, cxy, clab, counts, passes) device tensors.
        """
        t = self._torch
        st = self.settings
        if rgb.dim() == 3:
            rgb = rgb.unsqueeze(0)
        if (rgb.dtype != t.uint8 or not rgb.is_cuda or not rgb.is_contiguous()
                or tuple(rgb.shape[1:]) != (st.img_height, st.img_width, 3)):
            raise DimensionMismatchError(
                f"frames must be contiguous CUDA uint8 (B, {st.img_height}, {st.img_width}, 3), "
                f"got {tuple(rgb.shape)} {rgb.dtype}")
        dev = t.device("cuda", self.device)
        if rgb.device != dev:
            raise DimensionMismatchError(f"frames are on {rgb.device}, engine runs on {dev}")
        b = rgb.shape[0]
        if b < 1 or b > self.max_batch:
            raise DimensionMismatchError(f"batch {b} outside [1, {self.max_batch}] (max_batch)")
        if out is None:
            out = self.allocate_outputs(b)
        self._check_outputs(out, b)
        labels, cxy, clab, counts, passes = out
        s = stream if stream is not None else t.cuda.current_stream(self.device)
        _lib.check(self._lib.spx_engine_segment(
            self._h, ctypes.c_void_p(rgb.data_ptr()), b, ctypes.c_void_p(labels.data_ptr()),
            ctypes.c_void_p(cxy.data_ptr()), ctypes.c_void_p(clab.data_ptr()),
            ctypes.c_void_p(counts.data_ptr()), ctypes.c_void_p(passes.data_ptr()),
            ctypes.c_void_p(s.cuda_stream)), "segment")
        return out

    def _check_outputs(self, out, b):
        """Output tensors must hold (at least) `b` frames: the kernels write
        b frames' worth of results through raw pointers."""
        t = self._torch
        st = self.settings
        k = self.grid.num_clusters
        if not isinstance(out, (tuple, list)) or len(out) != 5:
            raise DimensionMismatchError("out must be (labels, cxy, clab, counts, passes)")
        dev = t.device("cuda", self.device)
        for name, a, shape, dt in (("labels", out[0], (st.img_height, st.img_width), t.int32),
                                   ("cxy", out[1], (k, 2), t.float64),
                                   ("clab", out[2], (k, 3), t.float64),
                                   ("counts", out[3], (k,), t.int64),
                                   ("passes", out[4], (), t.int32)):
            if (not isinstance(a, t.Tensor) or a.dtype != dt or a.device != dev
                    or not a.is_contiguous() or a.dim() != 1 + len(shape)
                    or tuple(a.shape[1:]) != shape or a.shape[0] < b):
                got = (tuple(a.shape), a.dtype, str(a.device)) if isinstance(a, t.Tensor) else type(a)
                raise DimensionMismatchError(
                    f"out {name} must be a contiguous {dt} tensor on {dev} of shape "
                    f"(>= {b}, {', '.join(map(str, shape))}), got {got}")

    def segment_host(self, rgb, labels=None, cxy=None, clab=None, counts=None, passes=None):
        """Segment host uint8 frames (B, H, W, 3) through the C ABI's host-buffer call.

        Inputs and outputs are numpy arrays (pinned memory is used as-is).
        Synchronous.  Returns (labels, cxy, clab, counts, passes).
        """
        st = self.settings
        rgb = np.ascontiguousarray(rgb, dtype=np.uint8)
        if rgb.ndim == 3:
            rgb = rgb[None]
        if rgb.shape[1:] != (st.img_height, st.img_width, 3):
            raise DimensionMismatchError(
                f"frame is {rgb.shape[2]}x{rgb.shape[1]}, engine expects "
                f"{st.img_width}x{st.img_height}")
        b = rgb.shape[0]
        k = self.grid.num_clusters
        if labels is None:
            labels = np.empty((b, st.img_height, st.img_width), dtype=np.int32)
        if cxy is None:
            cxy = np.empty((b, k, 2))
        if clab is None:
            clab = np.empty((b, k, 3))
        if counts is None:
            counts = np.empty((b, k), dtype=np.int64)
        if passes is None:
            passes = np.empty(b, dtype=np.int32)
        p = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        _lib.check(self._lib.spx_engine_segment_host(self._h, p(rgb), b, p(labels), p(cxy),
                                                     p(clab), p(counts), p(passes)), "segment")
        return labels, cxy, clab, counts, passes

    def submit_host(self, rgb, labels, cxy, clab, counts, passes):
        """Enqueue one batch of host frames without waiting (stream of batches).

        All arrays must be caller-owned numpy arrays (pinned for overlap) that
        stay alive and unread until `wait()`.  Consecutive submits share one
        H2D / compute / D2H pipeline.
        """
        st = self.settings
        if rgb.ndim != 4 or rgb.shape[1:] != (st.img_height, st.img_width, 3) or \
                rgb.dtype != np.uint8 or not rgb.flags.c_contiguous:
            raise DimensionMismatchError("submit_host needs contiguous uint8 (B, H, W, 3) frames")
        b = rgb.shape[0]
        k = self.grid.num_clusters
        for a, shape, dt in ((labels, (b, st.img_height, st.img_width), np.int32),
                             (cxy, (b, k, 2), np.float64), (clab, (b, k, 3), np.float64),
                             (counts, (b, k), np.int64), (passes, (b,), np.int32)):
            if a.shape != shape or a.dtype != dt or not a.flags.c_contiguous:
                raise ValueError(f"output {a.shape}/{a.dtype} does not match {shape}/{np.dtype(dt)}")
        self._pending.append((rgb, labels, cxy, clab, counts, passes))
        p = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        _lib.check(self._lib.spx_engine_submit_host(self._h, p(rgb), b, p(labels), p(cxy),
                                                    p(clab), p(counts), p(passes)), "submit")
        return int(self._lib.spx_engine_ticket(self._h))

    def wait_ticket(self, ticket):
        """Wait for the submission that returned `ticket` (and all before it)."""
        _lib.check(self._lib.spx_engine_wait_ticket(self._h, int(ticket)), "wait_ticket")

    def ticket_time(self, ticket):
        """Device time (seconds) of the submission that returned `ticket`;
        waits for that submission's compute only."""
        ms = ctypes.c_float()
        _lib.check(self._lib.spx_engine_ticket_time(self._h, int(ticket), ctypes.byref(ms)),
                   "ticket_time")
        return ms.value * 1e-3

    def set_host_chunk(self, frames):
        """Frames per H2D/compute/D2H pipeline chunk of the host-buffer path."""
        _lib.check(self._lib.spx_engine_set_host_chunk(self._h, int(frames)), "set_host_chunk")

    def set_lanes(self, lanes):
        """Concurrent sub-batches per call (0 = automatic: 1 below 4 frames,
        3 for calls of more than 64 frames under 24 Mpx, else 4).  Results do
        not depend on it."""
        _lib.check(self._lib.spx_engine_set_lanes(self._h, int(lanes)), "set_lanes")

    def last_lanes(self):
        return int(self._lib.spx_engine_last_lanes(self._h))

    def wait(self):
        """Wait for every submitted batch; their outputs are then valid."""
        _lib.check(self._lib.spx_engine_wait(self._h), "wait")
        self._pending.clear()

    def last_timing(self, max_updates=None):
        """Per-stage device times (seconds) of the last call, batch-wide
        (`max_updates`: keep only that many update passes and one more
        association, the passes a given frame ran)."""
        tb = self.__dict__.get("_timing_buf")
        if tb is None:
            t = _lib.SpxTiming()
            tb = self._timing_buf = (t, ctypes.byref(t))
        t, ref = tb
        rc = self._lib.spx_engine_timing(self._h, ref)
        if rc:
            _lib.check(rc, "timing")
        na, nu = t.n_associate, t.n_update
        if max_updates is not None:
            nu = min(nu, max_updates)
            na = min(na, max_updates + 1)
        ms = 1e-3
        return StageTiming(t.convert * ms, t.init * ms, t.perturb * ms,
                           tuple([v * ms for v in t.associate[:na]]),
                           tuple([v * ms for v in t.update[:nu]]),
                           t.connectivity * ms, t.total * ms)

    def last_launches(self):
        return int(self._lib.spx_engine_last_launches(self._h))

    @property
    def fused_path(self):
        """True when the engine runs the fused cell kernels (4 <= S <= 255)."""
        return bool(self._lib.spx_engine_fused_path(self._h))

    # ---- reference API ---------------------------------------------------------------

    def _check_frame(self, img):
        st = self.settings
        if (img.height, img.width) != (st.img_height, st.img_width):
            raise DimensionMismatchError(
                f"frame is {img.width}x{img.height}, engine expects "
                f"{st.img_width}x{st.img_height}")

    def _results(self, labels, cxy, clab, counts, passes, timing):
        out = []
        for i in range(labels.shape[0]):
            n_up = int(passes[i])
            tm = StageTiming(timing.convert, timing.init, timing.perturb,
                             timing.associate[:n_up + 1], timing.update[:n_up],
                             timing.connectivity, timing.total)
            out.append(SegResult(labels=LabelMap(labels[i]),
                                 spixel_map=SuperpixelMap(self.grid, cxy[i], clab[i], counts[i]),
                                 timing=tm))
        return out

    def _pinned_outputs(self, b):
        """Fresh result arrays for `b` frames carved from ONE pinned host block
        (torch's caching host allocator) in the engine's output layout, so the
        device results come back with a single D2H copy and need no copy-out.
        The block lives as long as the returned arrays do."""
        cache = self.__dict__.setdefault("_layouts", {})
        spec = cache.get(b)
        if spec is None:
            st = self.settings
            k = self.grid.num_clusters
            lay = (ctypes.c_int64 * 6)()
            _lib.check(self._lib.spx_engine_output_layout(self._h, b, lay), "output_layout")
            shapes = (((b, st.img_height, st.img_width), np.int32), ((b, k, 2), np.float64),
                      ((b, k, 3), np.float64), ((b, k), np.int64), ((b,), np.int32))
            spec = (int(lay[5]), [(int(lay[i]), int(np.prod(sh)) * np.dtype(dt).itemsize, sh,
                                   np.dtype(dt)) for i, (sh, dt) in enumerate(shapes)])
            cache[b] = spec
        total, parts = spec
        blk = self._torch.empty((total,), dtype=self._torch.uint8, pin_memory=True).numpy()
        return tuple(blk[o:o + n].view(dt).reshape(sh) for o, n, sh, dt in parts)

    def _pinned_input(self, b):
        """Engine-owned pinned staging for `b` input frames (grown on demand)."""
        st = self.settings
        buf = getattr(self, "_pin_in", None)
        if buf is None or buf.shape[0] < b:
            t = self._torch
            buf = t.empty((b, st.img_height, st.img_width, 3), dtype=t.uint8,
                          pin_memory=True).numpy()
            self._pin_in = buf
            self._pin_in_ptr = buf.__array_interface__["data"][0]
        return buf[:b]

    def perform_segmentation(self, img):
        """Run the full pipeline on one ImageRGB frame (engine.py:125-230).

        The frame is staged through an engine-owned pinned buffer and the
        results land in a fresh pinned block (one D2H); the call is
        synchronous, as the reference's."""
        self._check_frame(img)
        fast = self.__dict__.get("_ps_fast")
        if fast is None:
            fast = self._ps_fast = self._perform_prepare()
        pin0, pin_ptr, total, parts = fast
        np.copyto(pin0, img.data)
        blk = self._torch.empty((total,), dtype=self._torch.uint8, pin_memory=True).numpy()
        base = blk.__array_interface__["data"][0]
        rc = self._lib.spx_engine_segment_host(self._h, pin_ptr, 1, *(base + o for o, _, _ in parts))
        if rc:
            _lib.check(rc, "segment")
        # one frame's arrays straight on the block (they keep it alive)
        labels, cxy, clab, counts, passes = (np.ndarray(sh, dt, blk, o) for o, sh, dt in parts)
        tm = self.last_timing(max_updates=int(passes[0]))
        return SegResult(labels=LabelMap._trusted(labels),
                         spixel_map=SuperpixelMap._trusted(self.grid, cxy, clab, counts),
                         timing=tm)

    def _perform_prepare(self):
        """Per-engine constants of perform_segmentation: the pinned staging
        frame and its address, and the one-frame result block's layout."""
        pin = self._pinned_input(1)
        self._pinned_outputs(1)  # fills the layout cache
        total, parts = self._layouts[1]
        st = self.settings
        k = self.grid.num_clusters
        shapes = ((st.img_height, st.img_width), (k, 2), (k, 3), (k,), (1,))
        return (pin[0], self._pin_in_ptr, total,
                [(o, sh, dt) for (o, _, _, dt), sh in zip(parts, shapes)])

    def perform_segmentation_batch(self, imgs):
        """Segment a list of same-sized frames in batches of max_batch."""
        out = []
        for i, img in enumerate(imgs):
            try:
                self._check_frame(img)
            except DimensionMismatchError as exc:
                raise DimensionMismatchError(f"frame {i}: {exc}") from None
        for lo in range(0, len(imgs), self.max_batch):
            chunk = np.stack([im.data for im in imgs[lo:lo + self.max_batch]])
            res = self.segment_host(chunk)
            out.extend(self._results(*res, self.last_timing()))
        return out


def perform_segmentation(engine, img):
    """Functional form of SegEngine.perform_segmentation."""
    return engine.perform_segmentation(img)


def segment_stream(engine, imgs):
    """Yield one SegResult per frame, batching up to engine.max_batch frames.

    Batches go through the engine's host pipeline with two pinned buffer sets:
    batch i+1 is uploaded and segmented while batch i's results are returned,
    so the copies overlap the GPU work (engine.py:238-249 runs the batches one
    after another).  A frame of the wrong size aborts the stream with
    DimensionMismatchError naming its index, after the results of the frames
    before it.
    """
    import collections
    torch = engine._torch
    st, k, mb = engine.settings, engine.grid.num_clusters, engine.max_batch
    h, w = st.img_height, st.img_width

    def pinned(shape, dt):
        return torch.empty(shape, dtype=dt).pin_memory().numpy()

    sets = [None, None]
    inflight = collections.deque()

    def submit(frames, slot):
        if sets[slot] is None:
            sets[slot] = (pinned((mb, h, w, 3), torch.uint8), pinned((mb, h, w), torch.int32),
                          pinned((mb, k, 2), torch.float64), pinned((mb, k, 3), torch.float64),
                          pinned((mb, k), torch.int64), pinned((mb,), torch.int32))
        bufs = sets[slot]
        n = len(frames)
        for j, img in enumerate(frames):
            bufs[0][j] = img.data
        ticket = engine.submit_host(*(b[:n] for b in bufs))
        inflight.append((ticket, slot, n))

    def drain_one():
        ticket, slot, n = inflight.popleft()
        engine.wait_ticket(ticket)
        bufs = sets[slot]
        # This batch's own device time (engine.last_timing() would describe,
        # and wait for, the newest submission); per-stage times are not kept
        # per submission and read 0.
        total = engine.ticket_time(ticket)
        passes = bufs[5][:n]
        n_up = int(passes.max()) if n else 0
        tm = StageTiming(0.0, 0.0, 0.0, (0.0,) * (n_up + 1), (0.0,) * n_up, 0.0, total)
        # copies: the pinned set is reused by the next-but-one batch
        return engine._results(*(b[:n].copy() for b in bufs[1:]), tm)

    pending, slot = [], 0
    try:
        for i, img in enumerate(imgs):
            try:
                engine._check_frame(img)
            except DimensionMismatchError as exc:
                if pending:
                    submit(pending, slot)
                while inflight:
                    yield from drain_one()
                raise DimensionMismatchError(f"frame {i}: {exc}") from None
            pending.append(img)
            if len(pending) == mb:
                if len(inflight) == 2:
                    yield from drain_one()
                submit(pending, slot)
                slot ^= 1
                pending = []
        if pending:
            if len(inflight) == 2:
                yield from drain_one()
            submit(pending, slot)
        while inflight:
            yield from drain_one()
    finally:
        engine.wait()

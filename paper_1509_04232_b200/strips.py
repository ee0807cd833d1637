"""Row-strip segmentation of one large image across ranks.

Each rank owns a contiguous block of grid cell rows (`sharding.strip_plan`)
and runs the native strip engine (csrc/strips.cu) on its RGB window (own rows
plus one halo cell row above and below).  Per iteration neighbours exchange
boundary-cluster centres, boundary-cluster partial sums and S halo label rows;
the result is bit-identical to segmenting the whole image on one GPU.

Transports:
  * `DistComm`  -- torch.distributed point-to-point (NCCL over NVLink between
    GPUs; gloo works for CPU tensors in tests);
  * `LocalComm` -- several strips in one process (device copies), used to
    validate the decomposition on a single GPU.  Strips run one after another;
    no kernel ever waits on another strip.
"""

import ctypes

import numpy as np

from . import _lib, slic_core
from .connectivity import default_min_size
from .engine import _native_settings
from .errors import InvalidSettingsError
from .sharding import strip_plan

ACC_BYTES = 48  # sizeof(ClusterAcc)


def _p(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


class StripEngine:
    """One strip (cell rows [row_lo, row_hi)) of a large image on one device."""

    def __init__(self, settings, row_lo, row_hi, device=0):
        import torch
        self.torch = torch
        self.settings = settings
        self.grid = slic_core.compute_grid(settings)
        self.device = torch.device("cuda", device)
        self._st = _native_settings(settings, self.grid)
        lib = _lib.load()
        h = ctypes.c_void_p()
        _lib.check(lib.spx_strip_create(ctypes.byref(self._st), row_lo, row_hi, device,
                                        ctypes.byref(h)), "strip")
        self._h, self._lib = h, lib
        g = (ctypes.c_int64 * 6)()
        _lib.check(lib.spx_strip_geometry(h, g), "strip geometry")
        self.y0, self.hl, self.own_y0, self.own_y1, self.row_lo, self.row_hi = (int(v) for v in g)
        c, s, w = self.grid.ns_c, self.grid.s, settings.img_width
        dev = self.device
        self.has_up = row_lo > 0
        self.has_down = row_hi < self.grid.ns_r
        mk = lambda shape, dt: torch.zeros(shape, dtype=dt, device=dev)  # noqa: E731
        # send/recv buffers, index 0 = towards the upper neighbour, 1 = lower
        self.centres = [[mk((c * 5,), torch.float64) for _ in range(2)] for _ in range(2)]
        self.sums = [[mk((c * ACC_BYTES,), torch.uint8) for _ in range(2)] for _ in range(2)]
        self.labels = [[mk((s * w,), torch.int32) for _ in range(2)] for _ in range(2)]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                self._lib.spx_strip_destroy(h)
            except Exception:
                pass
            self._h = None

    def _stream(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream(self.device).cuda_stream)

    def _call(self, name, *args):
        _lib.check(getattr(self._lib, name)(self._h, *args, self._stream()), name)

    def _pair(self, bufs, send):
        i = 0 if send else 1
        up = bufs[0][i] if self.has_up else None
        down = bufs[1][i] if self.has_down else None
        return _p(up), _p(down)

    # kernel steps
    def begin(self, rgb_window):
        self._call("spx_strip_begin", _p(rgb_window))

    def associate(self, with_update):
        self._call("spx_strip_associate", int(with_update))

    def update(self):
        self._call("spx_strip_update")

    def pack(self, what):
        self._call(f"spx_strip_pack_{what}", *self._pair(getattr(self, what), True))

    def unpack(self, what):
        self._call(f"spx_strip_unpack_{what}", *self._pair(getattr(self, what), False))

    def finish(self):
        t = self.torch
        c = self.grid.ns_c
        n_own = self.row_hi - self.row_lo
        labels = t.empty((self.own_y1 - self.own_y0, self.settings.img_width), dtype=t.int32,
                         device=self.device)
        cxy = t.empty((n_own * c, 2), dtype=t.float64, device=self.device)
        clab = t.empty((n_own * c, 3), dtype=t.float64, device=self.device)
        counts = t.empty((n_own * c,), dtype=t.int64, device=self.device)
        self._call("spx_strip_finish", _p(labels), _p(cxy), _p(clab), _p(counts))
        return labels, cxy, clab, counts


class LocalComm:
    """Neighbour exchange between strips held by one process (device copies)."""

    def __init__(self, strips):
        self.strips = strips

    def exchange(self, what):
        for st in self.strips:
            st.pack(what)
        for i, st in enumerate(self.strips):
            bufs = getattr(st, what)
            if st.has_up:  # from the upper strip's "down" send buffer
                bufs[0][1].copy_(getattr(self.strips[i - 1], what)[1][0])
            if st.has_down:
                bufs[1][1].copy_(getattr(self.strips[i + 1], what)[0][0])
        for st in self.strips:
            st.unpack(what)


class DistComm:
    """Neighbour exchange between ranks with torch.distributed send/recv.

    Buffers are [[send_up, recv_up], [send_down, recv_down]].  With NCCL the
    device buffers go over NVLink directly; with gloo (CPU transport, used for
    functional tests) device buffers are staged through host memory.
    """

    def __init__(self, rank, world, group=None):
        self.rank, self.world, self.group = rank, world, group

    def exchange_buffers(self, bufs):
        import torch.distributed as dist
        if bufs[0][0].is_cuda and dist.get_backend(self.group) == "gloo":
            host = [[b.cpu() for b in pair] for pair in bufs]
            self._exchange(host)
            for pair, hpair in zip(bufs, host):
                pair[1].copy_(hpair[1])
            return
        self._exchange(bufs)

    def _exchange(self, bufs):
        import torch.distributed as dist
        ops = []
        if self.rank > 0:
            ops.append(dist.P2POp(dist.isend, bufs[0][0], self.rank - 1, self.group))
            ops.append(dist.P2POp(dist.irecv, bufs[0][1], self.rank - 1, self.group))
        if self.rank < self.world - 1:
            ops.append(dist.P2POp(dist.isend, bufs[1][0], self.rank + 1, self.group))
            ops.append(dist.P2POp(dist.irecv, bufs[1][1], self.rank + 1, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def exchange(self, strip, what):
        strip.pack(what)
        self.exchange_buffers(getattr(strip, what))
        strip.unpack(what)


def _run(strips, xchg):
    """The per-strip step sequence (identical for local and distributed runs)."""
    st = strips[0].settings
    xchg("centres")
    for _ in range(st.no_iters):
        for s in strips:
            s.associate(True)
        xchg("sums")
        xchg("labels")
        for s in strips:
            s.update()
        xchg("centres")
    for s in strips:
        s.associate(False)
    xchg("labels")


def check_strip_settings(settings):
    if settings.early_stop_threshold is not None:
        raise InvalidSettingsError("row strips do not support early stop")
    if settings.do_enforce_connectivity and settings.connectivity_mode.value == "strict":
        raise InvalidSettingsError("row strips support weak or no connectivity")


def segment_strips_local(settings, rgb, n_strips, device=0):
    """Segment one image as `n_strips` row strips in this process (validation path).

    Returns numpy (labels, centers_xy, centers_lab, num_pixels) for the whole
    image, assembled from the strips' own rows / clusters.
    """
    import torch
    check_strip_settings(settings)
    grid = slic_core.compute_grid(settings)
    plan = strip_plan(settings.img_height, grid.s, grid.ns_r, n_strips)
    strips = [StripEngine(settings, p.cell_row_lo, p.cell_row_hi, device) for p in plan
              if p.cell_row_hi > p.cell_row_lo]
    d_rgb = torch.from_numpy(np.ascontiguousarray(rgb, dtype=np.uint8)).to(strips[0].device)
    for s in strips:
        s.begin(d_rgb[s.y0:s.y0 + s.hl].contiguous())
    comm = LocalComm(strips)
    _run(strips, comm.exchange)
    outs = [s.finish() for s in strips]
    torch.cuda.synchronize(strips[0].device)
    labels = torch.cat([o[0] for o in outs]).cpu().numpy()
    cxy = torch.cat([o[1] for o in outs]).cpu().numpy()
    clab = torch.cat([o[2] for o in outs]).cpu().numpy()
    counts = torch.cat([o[3] for o in outs]).cpu().numpy()
    return labels, cxy, clab, counts


def segment_strip_rank(settings, rgb_window, rank, world, device, group=None):
    """One rank's share of a distributed row-strip segmentation.

    `rgb_window` is this rank's RGB window (see StripEngine.y0 / hl, or
    `strip_window(settings, rank, world)`).  Returns device tensors for the
    rank's own rows / clusters.
    """
    check_strip_settings(settings)
    grid = slic_core.compute_grid(settings)
    p = strip_plan(settings.img_height, grid.s, grid.ns_r, world)[rank]
    strip = StripEngine(settings, p.cell_row_lo, p.cell_row_hi, device)
    strip.begin(rgb_window)
    comm = DistComm(rank, world, group)
    _run([strip], lambda what: comm.exchange(strip, what))
    return strip.finish()


def strip_window(settings, rank, world):
    """Global pixel rows [y0, y1) of `rank`'s RGB input window."""
    grid = slic_core.compute_grid(settings)
    p = strip_plan(settings.img_height, grid.s, grid.ns_r, world)[rank]
    lo = max(p.cell_row_lo - 1, 0)
    hi = min(p.cell_row_hi + 1, grid.ns_r)
    return lo * grid.s, min(hi * grid.s, settings.img_height)


__all__ = ["StripEngine", "LocalComm", "DistComm", "segment_strips_local", "segment_strip_rank",
           "strip_window", "default_min_size"]

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
ALL, INTERIOR, BOUNDARY = 0, 1, 2


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

    # kernel steps; part: 0 all own rows, 1 interior, 2 boundary (spx.h)
    def begin(self, rgb_window):
        self._call("spx_strip_begin", _p(rgb_window))

    def associate(self, with_update, part=ALL):
        self._call("spx_strip_associate_part", int(with_update), int(part))

    def update(self, part=ALL):
        self._call("spx_strip_update_part", int(part))

    @property
    def own_clusters(self):
        return (self.row_hi - self.row_lo) * self.grid.ns_c

    def shift_local(self):
        """|new - old| of the own centres after an update (x, y per cluster)."""
        out = self.torch.empty((self.own_clusters * 2,), dtype=self.torch.float64,
                               device=self.device)
        self._call("spx_strip_shift_local", _p(out))
        return out

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


def pairwise_sum(x):
    """numpy's pairwise sum of a contiguous float64 device vector (spx_pairwise_sum),
    returned as a 1-element device tensor."""
    import torch
    out = torch.empty((1,), dtype=torch.float64, device=x.device)
    lib = _lib.load()
    _lib.check(lib.spx_pairwise_sum(_p(x), x.numel(), _p(out),
                                    ctypes.c_void_p(torch.cuda.current_stream(x.device).cuda_stream)),
               "pairwise_sum")
    return out


class LocalComm:
    """Neighbour exchange between strips held by one process (device copies).

    start() packs every strip's send buffers; finish() copies them to the
    neighbours' receive buffers and unpacks (the same schedule as DistComm,
    executed in order)."""

    def __init__(self, strips):
        self.strips = strips

    def start(self, whats):
        for what in whats:
            for st in self.strips:
                st.pack(what)
        return whats

    def finish(self, whats):
        for what in whats:
            for i, st in enumerate(self.strips):
                bufs = getattr(st, what)
                if st.has_up:  # from the upper strip's "down" send buffer
                    bufs[0][1].copy_(getattr(self.strips[i - 1], what)[1][0])
                if st.has_down:
                    bufs[1][1].copy_(getattr(self.strips[i + 1], what)[0][0])
            for st in self.strips:
                st.unpack(what)

    def exchange(self, what):
        self.finish(self.start([what]))

    def shift(self):
        """The whole image's centre shift (device scalar): the strips' own
        |delta| arrays concatenated in cluster order, pairwise-summed."""
        import torch
        return pairwise_sum(torch.cat([st.shift_local() for st in self.strips]))


class DistComm:
    """Neighbour exchange between ranks with torch.distributed send/recv.

    Buffers are [[send_up, recv_up], [send_down, recv_down]].  With NCCL the
    device buffers go over NVLink directly, and start() returns without
    waiting: the transfer runs on NCCL's stream while this rank's stream
    computes, and finish() makes the stream wait for it (Work.wait()) before
    unpacking.  With gloo (CPU transport, functional tests) device buffers
    are staged through host memory and the exchange completes in start().
    """

    def __init__(self, rank, world, strip, group=None):
        self.rank, self.world, self.strip, self.group = rank, world, strip, group

    def _ops(self, bufs):
        import torch.distributed as dist
        ops = []
        if self.rank > 0:
            ops.append(dist.P2POp(dist.isend, bufs[0][0], self.rank - 1, self.group))
            ops.append(dist.P2POp(dist.irecv, bufs[0][1], self.rank - 1, self.group))
        if self.rank < self.world - 1:
            ops.append(dist.P2POp(dist.isend, bufs[1][0], self.rank + 1, self.group))
            ops.append(dist.P2POp(dist.irecv, bufs[1][1], self.rank + 1, self.group))
        return ops

    def _gloo(self):
        import torch.distributed as dist
        return dist.get_backend(self.group) == "gloo"

    def start(self, whats):
        import torch.distributed as dist
        st = self.strip
        for what in whats:
            st.pack(what)
        works = []
        for what in whats:
            bufs = getattr(st, what)
            if bufs[0][0].is_cuda and self._gloo():
                host = [[b.cpu() for b in pair] for pair in bufs]
                ops = self._ops(host)
                if ops:
                    for w in dist.batch_isend_irecv(ops):
                        w.wait()
                for pair, hpair in zip(bufs, host):
                    pair[1].copy_(hpair[1])
                continue
            ops = self._ops(bufs)
            if ops:
                works.extend(dist.batch_isend_irecv(ops))
        return whats, works

    def finish(self, handle):
        whats, works = handle
        for w in works:
            w.wait()  # NCCL: the current stream waits; the host does not
        for what in whats:
            self.strip.unpack(what)

    def exchange(self, strip, what):
        self.finish(self.start([what]))

    def strict_labels(self, own):
        """Strict connectivity for row strips: the ranks' raw own-row labels
        are gathered on rank 0, which runs the whole-image pass, and each rank
        gets its rows back (gather + scatter of 4 B/px)."""
        import torch
        import torch.distributed as dist
        st = self.strip.settings
        g = self.strip.grid
        plan = strip_plan(st.img_height, g.s, g.ns_r, self.world)
        rows = [p.y_hi - p.y_lo for p in plan]
        m = max(rows) * st.img_width
        gloo = self._gloo()
        dev = own.device
        pad = torch.zeros((m,), dtype=torch.int32, device=dev)
        pad[:own.numel()] = own.reshape(-1)
        src = pad.cpu() if gloo else pad
        parts = [torch.empty_like(src) for _ in range(self.world)] if self.rank == 0 else None
        dist.gather(src, parts, dst=0, group=self.group)
        chunks = None
        if self.rank == 0:
            full = torch.cat([t[:r * st.img_width] for t, r in zip(parts, rows)]).to(dev)
            res = strict_whole_image(st, full.reshape(st.img_height, st.img_width)).reshape(-1)
            chunks, o = [], 0
            for r in rows:
                c = torch.zeros((m,), dtype=torch.int32, device=dev)
                c[:r * st.img_width] = res[o:o + r * st.img_width]
                o += r * st.img_width
                chunks.append(c.cpu() if gloo else c)
        mine = torch.empty_like(src)
        dist.scatter(mine, chunks, src=0, group=self.group)
        return mine.to(dev)[:own.numel()].reshape(own.shape)

    def shift(self):
        """The whole image's centre shift: every rank's own |delta| gathered in
        rank (= cluster) order, then the same pairwise sum on every rank."""
        import torch
        import torch.distributed as dist
        local = self.strip.shift_local()
        g = self.strip.grid
        sizes = [2 * (p.cell_row_hi - p.cell_row_lo) * g.ns_c
                 for p in strip_plan(self.strip.settings.img_height, g.s, g.ns_r, self.world)]
        m = max(sizes)
        pad = torch.zeros((m,), dtype=torch.float64, device=local.device)
        pad[:local.numel()] = local
        if self._gloo():
            parts = [torch.empty((m,), dtype=torch.float64) for _ in range(self.world)]
            dist.all_gather(parts, pad.cpu(), group=self.group)
            parts = [t.to(local.device) for t in parts]
        else:
            parts = [torch.empty_like(pad) for _ in range(self.world)]
            dist.all_gather(parts, pad, group=self.group)
        full = torch.cat([t[:n] for t, n in zip(parts, sizes)])
        return pairwise_sum(full)


def _run(strips, comm):
    """The per-strip step sequence (identical for local and distributed runs).

    Each exchange overlaps the compute that does not need it: the centres
    travel while the interior rows associate, the partial sums and label
    halos while the interior clusters update.  With early stop, the shift of
    every update (all clusters, numpy's pairwise order) decides on the host
    whether the next association is the last (engine.py:196-200)."""
    st = strips[0].settings
    thr = st.early_stop_threshold
    h = comm.start(["centres"])
    for _ in range(st.no_iters):
        for s in strips:
            s.associate(True, INTERIOR)
        comm.finish(h)
        for s in strips:
            s.associate(True, BOUNDARY)
        h = comm.start(["sums", "labels"])
        for s in strips:
            s.update(INTERIOR)
        comm.finish(h)
        for s in strips:
            s.update(BOUNDARY)
        stop = thr is not None and float(comm.shift().item()) < thr
        h = comm.start(["centres"])
        if stop:
            break
    for s in strips:
        s.associate(False, INTERIOR)
    comm.finish(h)
    for s in strips:
        s.associate(False, BOUNDARY)
    comm.finish(comm.start(["labels"]))


def check_strip_settings(settings):
    """Row strips take every setting the fused engine takes (S in [4, 255],
    ceil(3S / tile_len) <= 64); the native strip create reports the rest."""
    slic_core.compute_grid(settings)


def _strict(settings):
    return settings.do_enforce_connectivity and settings.connectivity_mode.value == "strict"


def strict_whole_image(settings, labels):
    """Strict connectivity (_core.pyx:359-461) over a whole image's raw labels
    (a device int32 tensor [H][W]): the scan-order component pass is global,
    so row strips gather their raw labels and run it once (spx_strict_fill)."""
    import torch
    g = slic_core.compute_grid(settings)
    min_size = settings.min_size if settings.min_size is not None else default_min_size(g.s)
    out = torch.empty_like(labels)
    lib = _lib.load()
    _lib.check(lib.spx_strict_fill(_p(labels), _p(out), labels.shape[0], labels.shape[1],
                                   int(min_size), ctypes.c_void_p(
                                       torch.cuda.current_stream(labels.device).cuda_stream)),
               "strict_fill")
    return out


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
    _run(strips, LocalComm(strips))
    outs = [s.finish() for s in strips]
    lab = torch.cat([o[0] for o in outs])
    if _strict(settings):
        lab = strict_whole_image(settings, lab)
    torch.cuda.synchronize(strips[0].device)
    labels = lab.cpu().numpy()
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
    comm = DistComm(rank, world, strip, group)
    _run([strip], comm)
    out = strip.finish()
    if _strict(settings):
        out = (comm.strict_labels(out[0]),) + tuple(out[1:])
    return out


def strip_window(settings, rank, world):
    """Global pixel rows [y0, y1) of `rank`'s RGB input window."""
    grid = slic_core.compute_grid(settings)
    p = strip_plan(settings.img_height, grid.s, grid.ns_r, world)[rank]
    lo = max(p.cell_row_lo - 1, 0)
    hi = min(p.cell_row_hi + 1, grid.ns_r)
    return lo * grid.s, min(hi * grid.s, settings.img_height)


__all__ = ["StripEngine", "LocalComm", "DistComm", "segment_strips_local", "segment_strip_rank",
           "strip_window", "pairwise_sum", "default_min_size"]

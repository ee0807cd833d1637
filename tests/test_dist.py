"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 host logic.

Frame sharding has no collective on the data path; the only collective is the
max-over-ranks timing reduction.  Row strips are checked for exact cover.
"""

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_1509_04232_b200.sharding import frame_shard, max_over_ranks, strip_plan


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_frames, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = frame_shard(n_frames, world, rank)
    elapsed = 1.0 + rank  # pretend rank r took 1+r seconds
    worst = max_over_ranks(elapsed)
    q.put((rank, lo, hi, worst))
    dist.destroy_process_group()


@pytest.mark.parametrize("n_frames", [512, 7])
def test_frame_shards_cover_and_max_reduce(n_frames):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_frames, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(world))
    covered = []
    for rank, lo, hi, worst in res:
        covered.extend(range(lo, hi))
        assert worst == float(world)  # max over ranks, not rank-local
    assert covered == list(range(n_frames))


def test_frame_shard_single_rank_identity():
    assert frame_shard(10, 1, 0) == (0, 10)
    assert max_over_ranks(3.5) == 3.5
    with pytest.raises(ValueError):
        frame_shard(10, 2, 2)


@pytest.mark.parametrize("h,s,world", [(16384, 16, 8), (480, 16, 3), (100, 7, 4), (5, 5, 2)])
def test_strip_plan_exact_cover(h, s, world):
    ns_r = -(-h // s)
    plan = strip_plan(h, s, ns_r, world)
    assert plan[0].cell_row_lo == 0 and plan[-1].cell_row_hi == ns_r
    assert plan[0].y_lo == 0 and plan[-1].y_hi == h
    for a, b in zip(plan, plan[1:]):
        assert a.cell_row_hi == b.cell_row_lo and a.y_hi == b.y_lo
    for st in plan:
        assert st.halo_lo == max(st.cell_row_lo - 1, 0)
        assert st.halo_hi == min(st.cell_row_hi + 1, ns_r)


def _strip_worker(rank, world, port, q):
    """DistComm moves [[send_up, recv_up], [send_down, recv_down]] between
    vertical neighbours (gloo, CPU tensors)."""
    import torch
    import torch.distributed as dist

    from paper_1509_04232_b200.strips import DistComm
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)

    class FakeStrip:  # the exchange only needs the buffers and pack / unpack
        def __init__(self):
            self.centres = [[torch.full((5,), 100.0 * rank + 1), torch.zeros(5)],
                            [torch.full((5,), 100.0 * rank + 2), torch.zeros(5)]]
            self.labels = [[torch.full((3,), 10.0 * rank + 3), torch.zeros(3)],
                           [torch.full((3,), 10.0 * rank + 4), torch.zeros(3)]]
            self.packed, self.unpacked = [], []

        def pack(self, what):
            self.packed.append(what)

        def unpack(self, what):
            self.unpacked.append(what)

    st = FakeStrip()
    comm = DistComm(rank, world, st)
    h = comm.start(["centres", "labels"])  # both exchanges in flight at once
    comm.finish(h)
    assert st.packed == ["centres", "labels"] and st.unpacked == ["centres", "labels"]
    q.put((rank, float(st.centres[0][1][0]), float(st.centres[1][1][0]),
           float(st.labels[0][1][0]), float(st.labels[1][1][0])))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_strip_neighbour_exchange(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_strip_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(world))
    for rank, from_up, from_down, lab_up, lab_down in res:
        # from_up = the upper rank's "send down" (100*(r-1)+2); from_down = lower's "send up"
        assert from_up == (100.0 * (rank - 1) + 2 if rank > 0 else 0.0)
        assert from_down == (100.0 * (rank + 1) + 1 if rank < world - 1 else 0.0)
        assert lab_up == (10.0 * (rank - 1) + 4 if rank > 0 else 0.0)
        assert lab_down == (10.0 * (rank + 1) + 3 if rank < world - 1 else 0.0)


def test_strip_schedule_overlaps_and_stops_early():
    """strips._run issues each exchange before the compute that does not need
    it and waits for it only before the compute that does; with early stop it
    ends after the first update whose shift is below the threshold, with one
    last association (engine.py:196-200).  Fake strips / comm record the
    order (no GPU)."""
    from paper_1509_04232_b200 import Settings
    from paper_1509_04232_b200.strips import BOUNDARY, INTERIOR, _run

    log = []

    class FakeStrip:
        def __init__(self, settings):
            self.settings = settings

        def associate(self, with_update, part):
            log.append(("assoc", with_update, "interior" if part == INTERIOR else "boundary"))

        def update(self, part):
            log.append(("update", "interior" if part == INTERIOR else "boundary"))

    class FakeComm:
        def __init__(self, shifts):
            self.shifts = list(shifts)

        def start(self, whats):
            log.append(("start", tuple(whats)))
            return tuple(whats)

        def finish(self, h):
            log.append(("finish", h))

        def shift(self):
            class T:
                def __init__(self, v):
                    self.v = v

                def item(self):
                    return self.v
            log.append(("shift",))
            return T(self.shifts.pop(0))

    st = Settings(img_width=64, img_height=64, spixel_size=8, no_iters=3)
    _run([FakeStrip(st)], FakeComm([]))
    one_iter = [("assoc", True, "interior"), ("finish", ("centres",)),
                ("assoc", True, "boundary"), ("start", ("sums", "labels")),
                ("update", "interior"), ("finish", ("sums", "labels")),
                ("update", "boundary"), ("start", ("centres",))]
    tail = [("assoc", False, "interior"), ("finish", ("centres",)),
            ("assoc", False, "boundary"), ("start", ("labels",)), ("finish", ("labels",))]
    assert log == [("start", ("centres",))] + one_iter * 3 + tail

    log.clear()
    st = Settings(img_width=64, img_height=64, spixel_size=8, no_iters=9,
                  early_stop_threshold=5.0)
    _run([FakeStrip(st)], FakeComm([9.0, 7.0, 4.0, 1.0]))
    with_shift = one_iter[:7] + [("shift",)] + one_iter[7:]
    # passes 1, 2 continue; pass 3's shift 4.0 < 5.0: its association is the last
    assert log == [("start", ("centres",))] + with_shift * 3 + tail

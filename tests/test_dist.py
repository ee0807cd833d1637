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

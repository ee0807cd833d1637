"""Multi-GPU work division (one process per GPU, torch.distributed plumbing).

Two decompositions, following SURVEY.md §8(e):

* frame sharding (C3: batches of frames): frames are independent, so each
  rank owns a contiguous range of the global batch and there is NO
  collective on the data path -- only the timing max-reduce of the bench.
* row strips (C5: one gigapixel image): each rank owns whole cell rows, so
  every cluster has exactly one owner; association of a strip needs the
  centres of one cell row above/below (halo), and the centre update needs
  the partial sums that neighbouring strips computed for the owner's
  boundary clusters.  `strip_plan` computes that geometry; the exchange is
  a fixed-order combine so the result is independent of the rank count.
"""

from dataclasses import dataclass


def frame_shard(n_frames, world, rank):
    """Contiguous [lo, hi) frame range of `rank` (same split as engine.band_bounds)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    return (rank * n_frames) // world, ((rank + 1) * n_frames) // world


@dataclass(frozen=True)
class Strip:
    rank: int
    cell_row_lo: int   # first owned cell row
    cell_row_hi: int   # one past the last owned cell row
    y_lo: int          # first owned pixel row
    y_hi: int          # one past the last owned pixel row
    halo_lo: int       # first cell row whose centres association reads
    halo_hi: int       # one past the last such cell row


def strip_plan(height, s, ns_r, world):
    """Split ns_r cell rows over `world` ranks in contiguous, S-aligned strips."""
    if world < 1:
        raise ValueError("world must be >= 1")
    plan = []
    for r in range(world):
        lo = (r * ns_r) // world
        hi = ((r + 1) * ns_r) // world
        plan.append(Strip(rank=r, cell_row_lo=lo, cell_row_hi=hi,
                          y_lo=min(lo * s, height), y_hi=min(hi * s, height),
                          halo_lo=max(lo - 1, 0), halo_hi=min(hi + 1, ns_r)))
    return plan


def max_over_ranks(value, device=None):
    """Max of a float over all ranks (identity without an initialised group)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())

"""Distributed row strips end to end: one process per strip (torchrun).

    torchrun --nproc-per-node N tools/strips_dist.py [--size 1024] [--check]

Each rank segments its strip of one synthetic image with the strip engine and
exchanges halos / partial sums with its neighbours through DistComm (NCCL on
one GPU per rank; SPX_STRIPS_BACKEND=gloo stages through host memory and lets
ranks share a GPU for a functional check).  Rank 0 gathers the strips and, with
--check, compares them bit for bit with the whole-image engine.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1509_04232_b200 as spx  # noqa: E402
from paper_1509_04232_b200.strips import segment_strip_rank, strip_window  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=1024)
    ap.add_argument("--s", type=int, default=16)
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--early-stop", type=float, default=None)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--strict", action="store_true")
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    backend = os.environ.get("SPX_STRIPS_BACKEND", "nccl")
    dev = local % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    dist.init_process_group(backend)
    n = a.size
    st = spx.Settings(img_width=n, img_height=n, spixel_size=a.s, no_iters=a.iters,
                      early_stop_threshold=a.early_stop,
                      connectivity_mode=(spx.ConnectivityMode.STRICT if a.strict
                                         else spx.ConnectivityMode.WEAK))
    rgb = np.random.default_rng(7).integers(0, 256, (n, n, 3), dtype=np.uint8)
    y0, y1 = strip_window(st, rank, world)
    window = torch.from_numpy(np.ascontiguousarray(rgb[y0:y1])).cuda(dev)
    labels, cxy, clab, counts = segment_strip_rank(st, window, rank, world, dev)
    torch.cuda.synchronize(dev)
    parts = [t.cpu() for t in (labels, cxy, clab, counts)]
    gathered = [None] * world
    dist.all_gather_object(gathered, parts)
    if rank == 0:
        L = torch.cat([g[0] for g in gathered]).numpy()
        C = torch.cat([g[2] for g in gathered]).numpy()
        X = torch.cat([g[1] for g in gathered]).numpy()
        N = torch.cat([g[3] for g in gathered]).numpy()
        msg = f"{world} strips of {n}x{n} (S={a.s}, {backend})"
        if a.check:
            res = spx.SegEngine(st, device=dev).perform_segmentation(spx.ImageRGB(rgb))
            ok = (np.array_equal(L, res.labels.data)
                  and C.tobytes() == res.spixel_map.centers_lab.tobytes()
                  and X.tobytes() == res.spixel_map.centers_xy.tobytes()
                  and np.array_equal(N, res.spixel_map.num_pixels))
            msg += f": bit-identical to the whole-image engine: {ok}"
            print(msg, flush=True)
            if not ok:
                sys.exit(1)
        else:
            print(msg, flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

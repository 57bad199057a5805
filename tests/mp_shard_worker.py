"""Worker for tests/test_gpu_multirank.py, launched by torchrun with N ranks
that may share one GPU: each rank owns a contiguous shard of the traces
(device generator rank range), the query summaries travel over a gloo process
group through psg_comm_init_host, and every rank writes its outputs to
<out>/rank<r>.npz; rank 0 also writes the single-context result over all
traces (<out>/single.npz)."""
from __future__ import annotations

import os
import sys

import numpy as np
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_03561_b200 import Q_ALL, Context, scenarios  # noqa: E402
from paper_2605_03561_b200 import dist as pdist  # noqa: E402

N_TRACES, N_PER_NODE, SITES = 40, 4, [2, 3, 4]


def run(ctx: Context, lo: int, hi: int, T: int) -> dict:
    node_of = np.arange(lo, hi) // N_PER_NODE
    n_nodes = N_TRACES // N_PER_NODE
    node = np.arange(n_nodes)
    ctx.set_nodes(node_of, n_nodes, 4000 + node // 4, node % 4)
    info = ctx.query(Q_ALL, t0=T // 4, t1=3 * T // 4, anchor=1, sites=SITES, top_k=4, z_min=-1e300)
    out = {f"w_{k}": v for k, v in ctx.window().items()}
    out.update({f"c_{k}": v for k, v in ctx.cube().items()})
    out.update({f"s_{k}": v for k, v in ctx.stats(1.0).items()})
    out.update({f"o_{k}": v for k, v in ctx.outliers(n_nodes).items()})
    out["info"] = np.array([info["n_kept"], info["n_kept_global"], info["min_iterations"],
                            info["worst_site"], info["n_outliers"]], np.int64)
    return out


def main(out_dir: str) -> None:
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    cfg = scenarios.iterative(N_TRACES, 9, n_kernels=6, seed=3, jitter=0.25)
    T = 0
    with Context(0) as single:  # to learn T (and, on rank 0, the reference run)
        single.generate_iterative(cfg)
        T = int(single.shard()["t_max"])
        if rank == 0:
            np.savez(os.path.join(out_dir, "single.npz"), **run(single, 0, N_TRACES, T))
    lo, hi = pdist.shard_range(N_TRACES, world, rank)
    with Context(0) as ctx:
        ctx.comm_init_host(world, rank, pdist.torch_reducer())
        ctx.generate_iterative(cfg, lo, hi)
        res = run(ctx, lo, hi, T)
        res["range"] = np.array([lo, hi], np.int64)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])

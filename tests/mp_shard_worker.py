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

from paper_2605_03561_b200 import ANCHOR_AUTO, Q_ALL, Context, scenarios  # noqa: E402
from paper_2605_03561_b200 import dist as pdist  # noqa: E402

N_TRACES, N_PER_NODE, SITES = 40, 4, [2, 3, 4]


def run(ctx: Context, lo: int, hi: int, T: int, anchor: int = 1) -> dict:
    node_of = np.arange(lo, hi) // N_PER_NODE
    n_nodes = N_TRACES // N_PER_NODE
    node = np.arange(n_nodes)
    ctx.set_nodes(node_of, n_nodes, 4000 + node // 4, node % 4)
    # twice: the second query runs speculatively (one host round trip, its
    # collectives in a different order) and must give the same results
    first = None
    for rep in range(2):
        info = ctx.query(Q_ALL, t0=T // 4, t1=3 * T // 4, anchor=anchor, sites=SITES, top_k=4, z_min=-1e300)
        got = {f"w_{k}": v for k, v in ctx.window().items()}
        got.update({f"c_{k}": v for k, v in ctx.cube().items()})
        if rep == 0:
            first = got
    for k, v in first.items():
        if v is not None:
            assert np.array_equal(v, got[k]), f"speculative re-run differs: {k}"
    out = {f"w_{k}": v for k, v in ctx.window().items()}
    out.update({f"c_{k}": v for k, v in ctx.cube().items()})
    out.update({f"s_{k}": v for k, v in ctx.stats(1.0).items()})
    out.update({f"o_{k}": v for k, v in ctx.outliers(n_nodes).items()})
    out["info"] = np.array([info["n_kept"], info["n_kept_global"], info["min_iterations"],
                            info["worst_site"], info["n_outliers"], info["anchor"]], np.int64)
    return out


def dup_traces():
    """N_TRACES traces of anchor(1) / kernels 2..4 / root(0) iterations; trace 3
    re-enters the anchor subtree on the timestamp it left it (a candidate the
    exact pass 1 drops): only the rank owning trace 3 sees the optimistic pass
    miss, and every rank must re-run with it."""
    parent = np.array([0xFFFFFFFF, 0, 1, 1, 1, 0], np.uint32)
    rng = np.random.default_rng(11)
    ts, cx, off, tend = [], [], [0], []
    for t in range(N_TRACES):
        now = int(rng.integers(0, 50))
        for it in range(12):
            cx.append(1); ts.append(now)
            if t == 3 and it == 5:                # leave and re-enter on the same timestamp
                cx.append(5); ts.append(now)
                cx.append(1); ts.append(now)
            for k in (2, 3, 4):
                cx.append(k); ts.append(now)
                now += int(rng.integers(10, 100))
            cx.append(5); ts.append(now)          # leave the subtree
            now += 7
            cx.append(0); ts.append(now)
            now += 3
        off.append(len(ts))
        tend.append(now + 5)
    body = np.zeros(len(ts) * 12, np.uint8)
    body.reshape(-1, 12)[:, :8] = np.array(ts, np.uint64).view(np.uint8).reshape(-1, 8)
    body.reshape(-1, 12)[:, 8:] = np.array(cx, np.uint32).view(np.uint8).reshape(-1, 4)
    return parent, body, np.array(off, np.uint64), np.array(tend, np.uint64)


def load_dup(ctx: Context, lo: int, hi: int) -> None:
    parent, body, off, tend = dup_traces()
    ctx.set_cct(parent)
    sub = body[int(off[lo]) * 12:int(off[hi]) * 12]
    ctx.load_aos(sub, off[lo:hi + 1] - off[lo], np.arange(lo, hi, dtype=np.uint32) + 1, tend[lo:hi])


def main(out_dir: str, mode: str = "gen") -> None:
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    if mode == "nccl":
        # one GPU per rank, the summaries over NCCL on device buffers
        # (psg_comm_init: the unique id travels over the gloo group)
        dev = int(os.environ.get("LOCAL_RANK", rank))
        cfg = scenarios.iterative(N_TRACES, 9, n_kernels=6, seed=3, jitter=0.25)
        with Context(dev) as single:
            single.generate_iterative(cfg)
            T = int(single.shard()["t_max"])
            if rank == 0:
                np.savez(os.path.join(out_dir, "single.npz"), **run(single, 0, N_TRACES, T))
        lo, hi = pdist.shard_range(N_TRACES, world, rank)
        uid = [Context.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        with Context(dev) as ctx:
            ctx.comm_init(world, rank, uid[0])
            ctx.generate_iterative(cfg, lo, hi)
            res = run(ctx, lo, hi, T)
            res["range"] = np.array([lo, hi], np.int64)
            np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
        dist.barrier()
        dist.destroy_process_group()
        return
    if mode == "dup":
        with Context(0) as single:
            load_dup(single, 0, N_TRACES)
            T = int(single.shard()["t_max"])
            if rank == 0:
                np.savez(os.path.join(out_dir, "single.npz"), **run(single, 0, N_TRACES, T))
        lo, hi = pdist.shard_range(N_TRACES, world, rank)
        with Context(0) as ctx:
            ctx.comm_init_host(world, rank, pdist.torch_reducer())
            load_dup(ctx, lo, hi)
            res = run(ctx, lo, hi, T)
            res["range"] = np.array([lo, hi], np.int64)
            np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
        dist.barrier()
        dist.destroy_process_group()
        return
    # "auto": PSG_ANCHOR_AUTO, the owner of the smallest profile id runs
    # suggest_anchor and every rank receives it; "auto_empty": the same with
    # the last rank holding no traces
    anchor = ANCHOR_AUTO if mode.startswith("auto") else 1
    cfg = scenarios.iterative(N_TRACES, 9, n_kernels=6, seed=3, jitter=0.25)
    T = 0
    with Context(0) as single:  # to learn T (and, on rank 0, the reference run)
        single.generate_iterative(cfg)
        T = int(single.shard()["t_max"])
        if rank == 0:
            np.savez(os.path.join(out_dir, "single.npz"), **run(single, 0, N_TRACES, T, anchor))
    if mode == "auto_empty":
        lo, hi = pdist.shard_range(N_TRACES, world - 1, rank) if rank < world - 1 else (N_TRACES, N_TRACES)
    else:
        lo, hi = pdist.shard_range(N_TRACES, world, rank)
    with Context(0) as ctx:
        ctx.comm_init_host(world, rank, pdist.torch_reducer())
        ctx.generate_iterative(cfg, lo, hi)
        res = run(ctx, lo, hi, T, anchor)
        res["range"] = np.array([lo, hi], np.int64)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "gen")

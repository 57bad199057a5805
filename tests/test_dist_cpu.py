"""CPU, world_size 2 over gloo: the host side of the rank-sharded path.

* dist.torch_reducer — the host reducer psg_comm_init_host calls — reduces
  uint64 / float64 buffers in place (sum, max, min);
* dist.shard_range / node_aligned_ranges partition the traces;
* the sharded decomposition the multi-GPU query relies on: per-shard exact
  sufficient statistics (per (iteration, node) sum, max, sum of squares and
  the global min iteration count), all-reduced, reproduce the single-process
  savings / CV of the oracle (pinned to the reference by test_oracle.py).
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2605_03561_b200 import dist as pdist
from tests.helpers import GOLDEN


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _stats_from_sums(S, M, Q, n_kept, K):
    """k_stats_finalize restated: per node avg_mean, avg_max, savings, total, across CV."""
    nn = S.shape[1]
    out = np.zeros((nn, 5))
    for n in range(nn):
        am = sum((S[k, n] / 1e9) / n_kept for k in range(K)) / K
        ax = sum(M[k, n] / 1e9 for k in range(K)) / K
        acr = sum(100.0 * np.sqrt(float(n_kept * int(Q[k, n]) - int(S[k, n]) ** 2)) / float(S[k, n])
                  for k in range(K)) / K
        out[n] = [am, ax, ax - am, (ax - am) * K, acr]
    return out


def _worker(rank, world, port, result_q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    red = pdist.torch_reducer()
    out = {}
    # 1. the reducer
    # the last column straddles 2^63: rank 0 sends ~0 (a "nothing" sentinel
    # in unsigned order), rank 1 sends 5 -- min / max must compare unsigned
    a = np.array([rank + 1, 10 * rank, 2**40 + rank, 2**64 - 1 if rank == 0 else 5], np.uint64)
    b, c = a.copy(), a.copy()
    red(a, "sum")
    red(b, "max")
    red(c, "min")
    f = np.array([0.5 * (rank + 1)], np.float64)
    red(f, "sum")
    out["reducer"] = (a.tolist(), b.tolist(), c.tolist(), f.tolist())
    # 2. sharded sufficient statistics of the gamess-like golden fixture
    with np.load(os.path.join(GOLDEN, "gamess_like.npz")) as z:
        g = {k: z[k] for k in z.files}
    n = len(g["pid"])
    lo, hi = pdist.shard_range(n, world, rank)
    e0, e1 = int(g["off"][lo]), int(g["off"][hi])
    sh = {"ts": g["ts"][e0:e1], "ctx": g["ctx"][e0:e1], "off": g["off"][lo:hi + 1] - g["off"][lo],
          "t_end": g["t_end"][lo:hi], "pid": g["pid"][lo:hi]}
    cb = oracle.cube(sh, g["parent"], 1)
    kept = cb["iter_counts"][cb["iter_counts"] > 0]
    nn = len(cb["node_ids"])
    kk = np.array([kept.min() if len(kept) else 2**63 - 1, len(kept)], np.uint64)
    mn = kk[:1].copy()
    red(mn, "min")
    cnt = kk[1:].copy()
    red(cnt, "sum")
    K = int(mn[0])
    S = np.zeros((K, nn), np.uint64)
    M = np.zeros((K, nn), np.uint64)
    Q = np.zeros((K, nn), np.uint64)
    for t, it in enumerate(kept):
        base = int(cb["block_offset"][t])
        v = cb["incl"][base:base + K * nn].reshape(K, nn).astype(np.uint64)
        S += v
        M = np.maximum(M, v)
        Q += v * v
    red(S, "sum")
    red(M, "max")
    red(Q, "sum")
    out["merged"] = _stats_from_sums(S, M, Q, int(cnt[0]), K)
    result_q.put((rank, out))
    dist.destroy_process_group()


def test_shard_ranges_partition():
    for n in (0, 1, 7, 100):
        for world in (1, 2, 3, 8):
            rs = [pdist.shard_range(n, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            assert max(h - l for l, h in rs) - min(h - l for l, h in rs) <= 1
    node = np.repeat(np.arange(10), [3, 1, 4, 1, 5, 9, 2, 6, 5, 3])
    rs = pdist.node_aligned_ranges(node, 4)
    assert rs[0][0] == 0 and rs[-1][1] == len(node)
    for lo, hi in rs[1:]:
        assert lo == 0 or node[lo] != node[lo - 1]  # edges on node boundaries
    with pytest.raises(ValueError):
        pdist.node_aligned_ranges(node[::-1], 2)


def test_gloo_two_ranks_merge_equals_single_process():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a, b, c, f = res[0]["reducer"]
    assert a == [3, 10, 2 * 2**40 + 1, 4] and b == [2, 10, 2**40 + 1, 2**64 - 1]
    assert c == [1, 0, 2**40, 5]
    assert f == [1.5]
    # the merged sufficient statistics equal the oracle over all traces
    with np.load(os.path.join(GOLDEN, "gamess_like.npz")) as z:
        g = {k: z[k] for k in z.files}
    full = oracle.cube({k: g[k] for k in ("ts", "ctx", "off", "t_end", "pid")}, g["parent"], 1)
    for r in range(world):
        m = res[r]["merged"]
        for npos in range(len(full["node_ids"])):
            want, ok = oracle.node_stats(full, npos)
            got = m[npos]
            assert np.allclose(got[:4], want[:4], rtol=1e-9, atol=0), (npos, got, want)
            if ok:
                assert abs(got[4] - want[4]) <= 1e-9 * abs(want[4]) + 1e-9

"""The query's host round trips and the narrow ctx mirror.

* A query on traces an earlier query has sized runs every kernel back to back
  and synchronises once (the device status block, psg_capi.cu); a miss of
  its speculative capacities (a larger anchor subtree, a larger K, a pass-1
  region overflow) re-runs it with the host sizing each step.  Results are
  the oracle's either way.
* Pass 1 reads a 1-byte preorder mirror of the ctx words when every ctx <
  256 (SIMD subtree membership); PSG_NO_CTX8=1 and trees of more than 256
  contexts take the 4-byte path.  Both are bit-exact against the oracle."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from paper_2605_03561_b200 import Q_ALL, Q_CUBE, Q_STATS, scenarios
from tests.helpers import random_cct, random_traces, to_aos
from tests.test_gpu_parity import WINDOW_KEYS, check_cube, check_window

pytestmark = pytest.mark.gpu


def _cube_equal(ctx, o):
    g = ctx.cube()
    for k in ("node_ids", "iter_counts", "block_offset", "incl", "excl", "gap_incl", "gap_excl"):
        assert np.array_equal(g[k], o[k]), f"cube {k}"


def test_repeated_query_synchronises_once(gpu_ctx_factory):
    ctx = gpu_ctx_factory()
    cfg = scenarios.iterative(96, 14, n_kernels=9, seed=3)
    ctx.generate_iterative(cfg)
    tr = ctx.traces()
    parent = np.array([0xFFFFFFFF, 0] + [1] * 9 + [0], np.uint32)
    node = np.arange(96) // 8
    ctx.set_nodes(node, 12, 4000 + node // 4, node % 4)
    T = int(tr["t_end"].max())
    ow = oracle.window(tr, parent, T // 4, 3 * T // 4)
    oc = oracle.cube(tr, parent, 1)
    syncs = []
    for _ in range(3):
        info = ctx.query(Q_ALL, t0=T // 4, t1=3 * T // 4, anchor=1, sites=[2, 3, 4], top_k=4, z_min=-1e9)
        syncs.append(info["host_syncs"])
        w = ctx.window()
        for k in WINDOW_KEYS:
            assert np.array_equal(w[k], ow[k]), f"window {k}"
        _cube_equal(ctx, oc)
        assert info["n_kept"] == 96 and info["min_iterations"] == oc["iter_counts"].min()
        assert info["n_outliers"] == 4
    assert syncs[0] > 1, syncs  # the first query after the load sizes the buffers
    assert syncs[1] == 1 and syncs[2] == 1, syncs


def test_speculative_capacity_miss_reruns(gpu_ctx_factory):
    """The anchor with the smallest cube sizes the buffers; the one with the
    largest then misses the speculative cube / excl capacities and re-runs
    with exact sizes."""
    rng = np.random.default_rng(7)
    ctx = gpu_ctx_factory()
    n_ctx = 30
    parent = random_cct(rng, n_ctx)
    tr = random_traces(rng, 40, n_ctx, 3000, dup_prob=0.2)
    ctx.set_cct(parent)
    ctx.load_aos(to_aos(tr), tr["off"], tr["pid"], tr["t_end"])
    cubes = {a: oracle.cube(tr, parent, a) for a in range(n_ctx)}
    cells = {a: int(len(o["incl"])) for a, o in cubes.items() if len(o["incl"])}
    lo, hi = min(cells, key=cells.get), max(cells, key=cells.get)
    for anchor in (lo, hi, lo):
        info = ctx.query(Q_CUBE | Q_STATS, anchor=anchor)
        _cube_equal(ctx, cubes[anchor])
        if anchor == hi and cells[hi] > 2 * cells[lo]:
            assert info["host_syncs"] > 1  # the speculative run missed and re-ran


def test_pass1_region_overflow_under_speculation(gpu_ctx_factory):
    """A query with one boundary per trace sizes the buffers; on the same
    traces an anchor with a boundary every other event then overflows pass
    1's default regions (n/32 + 32) inside a speculative query, which flags
    it and re-runs."""
    ctx = gpu_ctx_factory()
    parent = np.array([0xFFFFFFFF, 0, 0], np.uint32)
    n_tr, n_ev = 6, 4000
    ts = np.concatenate([np.arange(n_ev, dtype=np.uint64) * 10 for _ in range(n_tr)])
    cx = np.tile(np.array([1, 2], np.uint32), n_tr * n_ev // 2)
    tr = {"ts": ts, "ctx": cx, "off": np.arange(n_tr + 1, dtype=np.uint64) * n_ev,
          "t_end": np.full(n_tr, 10 * n_ev, np.uint64), "pid": np.arange(1, n_tr + 1, dtype=np.uint32)}
    ctx.set_cct(parent)
    ctx.load_aos(to_aos(tr), tr["off"], tr["pid"], tr["t_end"])
    ctx.query(Q_CUBE | Q_STATS, anchor=0)  # the whole tree: one boundary per trace
    _cube_equal(ctx, oracle.cube(tr, parent, 0))
    o = oracle.cube(tr, parent, 1)
    assert int(o["iter_counts"][0]) >= n_ev // 2 - 1
    for _ in range(2):
        info = ctx.query(Q_CUBE | Q_STATS, anchor=1)
        _cube_equal(ctx, o)
    assert info["host_syncs"] == 1


@pytest.mark.parametrize("seed", range(3))
def test_pass1_without_ctx8_mirror(gpu_ctx_factory, monkeypatch, seed):
    monkeypatch.setenv("PSG_NO_CTX8", "1")
    rng = np.random.default_rng(100 + seed)
    ctx = gpu_ctx_factory()
    n_ctx = int(rng.integers(3, 40))
    parent = random_cct(rng, n_ctx)
    tr = random_traces(rng, 30, n_ctx, 2000, dup_prob=0.4)
    ctx.set_cct(parent)
    ctx.load_aos(to_aos(tr), tr["off"], tr["pid"], tr["t_end"])
    for anchor in sorted({0, 1, n_ctx - 1}):
        check_cube(ctx, tr, parent, anchor)


def test_more_than_256_contexts(gpu_ctx_factory):
    """n_ctx > 256: no narrow mirror; pass 1 reads the 4-byte ctx words with
    the membership table in shared memory."""
    rng = np.random.default_rng(5)
    ctx = gpu_ctx_factory()
    n_ctx = 700
    parent = random_cct(rng, n_ctx)
    tr = random_traces(rng, 12, n_ctx, 5000, dup_prob=0.2, ctx_pool=n_ctx)
    ctx.set_cct(parent)
    ctx.load_aos(to_aos(tr), tr["off"], tr["pid"], tr["t_end"])
    T = int(tr["t_end"].max())
    check_window(ctx, tr, parent, T // 5, 4 * T // 5)
    for anchor in (0, 1, 3):
        check_cube(ctx, tr, parent, anchor, stats=False)


def test_cct_change_after_load_rebuilds_mirror(gpu_ctx_factory):
    """The mirror holds preorder positions of the tree: a new tree on the same
    traces rebuilds it."""
    rng = np.random.default_rng(11)
    ctx = gpu_ctx_factory()
    n_ctx = 20
    p1, p2 = random_cct(rng, n_ctx), random_cct(rng, n_ctx)
    tr = random_traces(rng, 25, n_ctx, 1500, dup_prob=0.3)
    ctx.set_cct(p1)
    ctx.load_aos(to_aos(tr), tr["off"], tr["pid"], tr["t_end"])
    check_cube(ctx, tr, p1, 1)
    ctx.set_cct(p2)
    for anchor in (1, 2):
        check_cube(ctx, tr, p2, anchor)

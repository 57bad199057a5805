"""Work units (intra-trace split, SURVEY.md §5 "long-context"): pass 2 splits
traces longer than the unit size across warps, snapping each unit to chunk
starts and merging the window and within-rank sums of a split trace with
atomics.  The reference runs one thread per trace (itermodel.cpp:276); the
results must not depend on the split: bit-exact against the oracle and the
unsplit run, for any unit size."""
from __future__ import annotations

import time

import numpy as np
import pytest

import oracle
from paper_2605_03561_b200 import Q_ALL, Q_CUBE, Q_STATS, Q_WINDOW, scenarios
from tests.helpers import random_cct, random_traces, to_aos
from tests.test_gpu_parity import WINDOW_KEYS, check_cube, check_window

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("unit", [37, 300])
@pytest.mark.parametrize("seed", range(3))
def test_units_random_traces(gpu_ctx_factory, monkeypatch, seed, unit):
    """Random CCTs and traces (equal timestamps, repeated contexts, empty
    traces), every trace longer than `unit` events split: GPU == oracle."""
    monkeypatch.setenv("PSG_UNIT_EVENTS", str(unit))
    rng = np.random.default_rng(100 + seed)
    ctx = gpu_ctx_factory()
    n_ctx = int(rng.integers(3, 30))
    parent = random_cct(rng, n_ctx)
    tr = random_traces(rng, int(rng.integers(3, 25)), n_ctx, int(rng.integers(200, 3000)),
                       ctx_pool=int(rng.integers(2, n_ctx + 1)), dup_prob=float(rng.random()) * 0.5)
    ctx.set_cct(parent)
    ctx.load_aos(to_aos(tr), tr["off"], tr["pid"], tr["t_end"])
    T = int(tr["t_end"].max())
    for t0, t1 in ((0, T + 1), (T // 3, 2 * T // 3), (T // 5, T // 5 + 7)):
        check_window(ctx, tr, parent, t0, t1)
    for anchor in sorted({1, int(rng.integers(0, n_ctx))}):
        check_cube(ctx, tr, parent, anchor)


def _query_all(ctx, T, flags=Q_ALL):
    info = ctx.query(flags, t0=T // 4, t1=3 * T // 4, anchor=1, sites=[2, 3], top_k=3)
    out = {"info": info, "window": ctx.window(), "carry": ctx.carry(), "cube": ctx.cube(),
           "stats": ctx.stats(1.0)}
    return out


@pytest.mark.parametrize("unit", [500, 4096])
def test_units_iterative_equal_unsplit(gpu_ctx_factory, monkeypatch, unit):
    """The iterative generator (anchor subtree, many chunks per trace): the
    split query equals the unsplit one in every output, and the oracle."""
    ctx = gpu_ctx_factory()
    cfg = scenarios.iterative(24, 120, n_kernels=10, seed=7)
    ctx.generate_iterative(cfg)
    node = np.arange(24) // 4
    ctx.set_nodes(node, 6, 4000 + node // 2, node % 2)
    T = int(ctx.traces()["t_end"].max())
    monkeypatch.setenv("PSG_UNIT_EVENTS", str(1 << 40))
    ref = _query_all(ctx, T)
    monkeypatch.setenv("PSG_UNIT_EVENTS", str(unit))
    got = _query_all(ctx, T)
    for k in WINDOW_KEYS:
        assert np.array_equal(got["window"][k], ref["window"][k]), k
    for k in ("has", "ts", "ctx"):
        assert np.array_equal(got["carry"][k], ref["carry"][k]), k
    for k in ("iter_counts", "block_offset", "incl", "excl", "gap_incl", "gap_excl"):
        assert np.array_equal(got["cube"][k], ref["cube"][k]), k
    for k in ("savings", "summary", "cv", "cv_ok"):
        assert np.array_equal(got["stats"][k], ref["stats"][k]), k
    tr = ctx.traces()
    parent = np.array([0xFFFFFFFF, 0] + [1] * 10 + [0], np.uint32)
    o = oracle.cube(tr, parent, 1)
    for k in ("iter_counts", "incl", "excl", "gap_incl", "gap_excl"):
        assert np.array_equal(got["cube"][k], o[k]), k


def _long_and_short(rng, n_long, n_short, short_events):
    """One iterative trace of n_long events among n_short short ones: ctx 1 is
    the anchor, 2..9 its kernels, 10 a copy under the root; zero-length
    segments on anchor / root events like the reference generator."""
    per_it = [1] + list(range(2, 10)) + [10, 0]
    ts_all, cx_all, off, t_end = [], [], [0], []
    for n in [n_long] + [short_events] * n_short:
        reps = n // len(per_it) + 1
        cx = np.tile(np.array(per_it, np.uint32), reps)[:n]
        steps = rng.integers(1, 2000, size=n).astype(np.uint64)
        steps[(cx == 1) | (cx == 0)] = 0
        ts = np.cumsum(steps, dtype=np.uint64) + np.uint64(rng.integers(0, 100))
        ts_all.append(ts)
        cx_all.append(cx)
        off.append(off[-1] + n)
        t_end.append(int(ts[-1]) + 1000)
    parent = np.array([0xFFFFFFFF, 0] + [1] * 8 + [0], np.uint32)
    return {"ts": np.concatenate(ts_all), "ctx": np.concatenate(cx_all), "off": np.array(off, np.uint64),
            "t_end": np.array(t_end, np.uint64),
            "pid": np.arange(1, n_short + 2, dtype=np.uint32)}, parent


def test_one_long_trace_among_short(gpu_ctx_factory, monkeypatch):
    """One 20M-event trace among 1,000 short ones (the skewed input of VERDICT
    r1 #6): the default plan splits the long trace across the machine; window,
    cube and statistics stay bit-exact against the oracle and the unsplit run,
    and the split query is faster."""
    rng = np.random.default_rng(2026)
    tr, parent = _long_and_short(rng, 20_000_000, 1000, 2000)
    ctx = gpu_ctx_factory()
    ctx.set_cct(parent)
    ctx.load_aos(to_aos(tr), tr["off"], tr["pid"], tr["t_end"])
    T = int(tr["t_end"].max())
    t0, t1 = T // 4, 3 * T // 4

    def run():
        ctx.query(Q_WINDOW | Q_CUBE | Q_STATS, t0=t0, t1=t1, anchor=1)
        ms = min(ctx.query(Q_WINDOW | Q_CUBE | Q_STATS, t0=t0, t1=t1, anchor=1)["ms_main"] for _ in range(3))
        return ms, ctx.window(), ctx.cube(), ctx.stats(1.0)

    monkeypatch.delenv("PSG_UNIT_EVENTS", raising=False)
    ms_split, w, cb, st = run()
    monkeypatch.setenv("PSG_UNIT_EVENTS", str(1 << 40))
    ms_whole, w1, cb1, st1 = run()
    for k in WINDOW_KEYS:
        assert np.array_equal(w[k], w1[k]), k
    for k in ("iter_counts", "incl", "excl", "gap_incl", "gap_excl"):
        assert np.array_equal(cb[k], cb1[k]), k
    for k in ("savings", "cv", "cv_ok"):
        assert np.array_equal(st[k], st1[k]), k
    ow = oracle.window(tr, parent, t0, t1)
    for k in WINDOW_KEYS:
        assert np.array_equal(w[k], ow[k]), k
    oc = oracle.cube(tr, parent, 1)
    for k in ("iter_counts", "incl", "excl", "gap_incl", "gap_excl"):
        assert np.array_equal(cb[k], oc[k]), k
    print(f"long trace: k_trace_query {ms_split:.3f} ms split vs {ms_whole:.3f} ms on one warp")
    assert ms_split < ms_whole / 4

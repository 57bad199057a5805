"""The sparse window path (psg_sparse.cu): calling-context trees too large for
the fused kernel's per-warp window records (the paper's AMG run has 97,833
contexts), or PSG_Q_SPARSE.

Bar: the group_aggregate rows (count > 0) and the rematerialize rows (incl or
excl nonzero) equal, row for row and in (trace, ctx) order, the oracle's dense
result compacted, the unmodified reference's own ingest_traces +
group_aggregate + rematerialize (oracle/_ref), and the dense path's
rows on the same inputs; the cube of a large tree (global column table) equals
the oracle's tri_model."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from paper_2605_03561_b200 import Q_CLAMP_TEND, Q_CUBE, Q_OUTLIERS, Q_SPARSE, Q_STATS, Q_WINDOW, PsgError
from tests.helpers import assert_rel, random_cct, random_traces, to_aos
from tests.test_gpu_parity import check_cube

pytestmark = pytest.mark.gpu

GROUP_KEYS = ("count", "sum", "min", "max", "mean")


def dense_to_rows(o: dict) -> tuple[dict, dict]:
    """The oracle's dense [trace][ctx] window as (groups, remat) rows, (trace, ctx) order."""
    ti, ci = np.nonzero(o["count"] > 0)
    groups = {"trace": ti.astype(np.uint32), "ctx": ci.astype(np.uint32)}
    groups.update({k: o[k][ti, ci] for k in GROUP_KEYS})
    ti, ci = np.nonzero((o["incl"] != 0) | (o["excl"] != 0))
    remat = {"trace": ti.astype(np.uint32), "ctx": ci.astype(np.uint32), "incl": o["incl"][ti, ci],
             "excl": o["excl"][ti, ci]}
    return groups, remat


def check_rows(ctx, o, what):
    gg, gr = ctx.window_groups(), ctx.remat_rows()
    og, orr = dense_to_rows(o)
    for k in og:
        assert np.array_equal(gg[k], og[k]), f"{what}: groups {k}"
    for k in orr:
        assert np.array_equal(gr[k], orr[k]), f"{what}: remat {k}"
    c = ctx.carry()
    for k in ("has", "ts", "ctx"):
        assert np.array_equal(c[k], o["carry"][k]), f"{what}: carry {k}"


@pytest.mark.parametrize("seed", range(4))
def test_sparse_equals_dense_and_oracle(gpu_ctx_factory, seed):
    rng = np.random.default_rng(300 + seed)
    ctx = gpu_ctx_factory()
    n_ctx = int(rng.integers(3, 60))
    parent = random_cct(rng, n_ctx)
    tr = random_traces(rng, int(rng.integers(1, 50)), n_ctx, int(rng.integers(1, 3000)),
                       dup_prob=float(rng.random()) * 0.5)
    ctx.set_cct(parent)
    ctx.load_aos(to_aos(tr), tr["off"], tr["pid"], tr["t_end"])
    T = int(tr["t_end"].max()) if len(tr["t_end"]) else 10
    for t0, t1, clamp in ((0, T + 1, False), (T // 3, 2 * T // 3, False), (T // 2, T // 2, False),
                          (T // 4, 2 * T, True), (T + 5, T + 9, False)):
        o = oracle.window(tr, parent, t0, t1, clamp_tend=clamp)
        fl = Q_WINDOW | (Q_CLAMP_TEND if clamp else 0)
        info = ctx.query(fl | Q_SPARSE, t0=t0, t1=t1)
        assert info["window_sparse"] == 1
        check_rows(ctx, o, f"sparse [{t0},{t1})")
        assert info["n_window_groups"] == int((o["count"] > 0).sum())
        with pytest.raises(PsgError):
            ctx.window()  # a sparse window has no dense copy-out
        info = ctx.query(fl, t0=t0, t1=t1)  # dense, copied out through the same accessors
        assert info["window_sparse"] == 0
        check_rows(ctx, o, f"dense [{t0},{t1})")


def _large_tree(rng, n_ctx):
    """A random tree of n_ctx contexts with a bounded depth (AMG-like: wide)."""
    parent = np.empty(n_ctx, np.uint32)
    parent[0] = 0xFFFFFFFF
    parent[1:] = (rng.random(n_ctx - 1) * np.arange(1, n_ctx) ** 0.9).astype(np.uint32)
    return parent


def test_large_tree_100k_contexts_against_reference(gpu_ctx_factory, tmp_path):
    """100,000 contexts: the window takes the sparse path by itself (the per-warp
    records do not fit); rows equal the oracle and the unmodified reference."""
    rng = np.random.default_rng(17)
    ctx = gpu_ctx_factory()
    n_ctx = 100_000
    parent = _large_tree(rng, n_ctx)
    tr = random_traces(rng, 24, n_ctx, 20_000, dup_prob=0.2, ctx_pool=n_ctx)
    ctx.set_cct(parent)
    ctx.load_aos(to_aos(tr), tr["off"], tr["pid"], tr["t_end"])
    T = int(tr["t_end"].max())
    d = str(tmp_path / "db")
    oracle.ref_write_traces(tr, parent, d)
    row = {int(p): i for i, p in enumerate(tr["pid"])}
    for t0, t1 in ((T // 4, 3 * T // 4), (0, T + 1)):
        info = ctx.query(Q_WINDOW, t0=t0, t1=t1)
        assert info["window_sparse"] == 1
        check_rows(ctx, oracle.window(tr, parent, t0, t1), f"100k [{t0},{t1})")
        r = oracle.ref_window(d, t0, t1)
        g, rm = ctx.window_groups(), ctx.remat_rows()
        assert np.array_equal(g["trace"], np.array([row[int(p)] for p in r["wa_pid"]], np.uint32))
        assert np.array_equal(g["ctx"], r["wa_ctx"].astype(np.uint32))
        for k in GROUP_KEYS:
            assert np.array_equal(g[k], r[f"wa_{k}"]), f"reference group_aggregate {k}"
        assert np.array_equal(rm["trace"], np.array([row[int(p)] for p in r["rm_pid"]], np.uint32))
        assert np.array_equal(rm["ctx"], r["rm_ctx"])
        assert np.array_equal(rm["incl"], r["rm_incl"]) and np.array_equal(rm["excl"], r["rm_excl"])


def test_amg_shape_98k_distinct_contexts_per_trace(gpu_ctx_factory, monkeypatch):
    """Traces that each touch ~98k distinct contexts (a permutation sweep per
    trace), in small batches of traces (the scratch bound is exercised by the
    row budget of one batch)."""
    monkeypatch.setenv("PSG_SPARSE_ROW_BUDGET", "150000")  # one trace per batch
    rng = np.random.default_rng(23)
    ctx = gpu_ctx_factory()
    n_ctx = 97_833
    parent = _large_tree(rng, n_ctx)
    ts, cx, off, tend = [], [], [0], []
    for t in range(4):
        perm = rng.permutation(n_ctx).astype(np.uint32)
        n = int(n_ctx * 1.2)
        c = np.concatenate([perm, perm[: n - n_ctx]])
        s = np.cumsum(rng.integers(0, 40, n)).astype(np.uint64) + np.uint64(rng.integers(0, 100))
        ts.append(s)
        cx.append(c)
        off.append(off[-1] + n)
        tend.append(int(s[-1]) + 7)
    tr = {"ts": np.concatenate(ts), "ctx": np.concatenate(cx), "off": np.array(off, np.uint64),
          "t_end": np.array(tend, np.uint64), "pid": np.arange(1, 5, dtype=np.uint32)}
    ctx.set_cct(parent)
    ctx.load_aos(to_aos(tr), tr["off"], tr["pid"], tr["t_end"])
    T = int(tr["t_end"].max())
    info = ctx.query(Q_WINDOW, t0=0, t1=T + 1)
    o = oracle.window(tr, parent, 0, T + 1)
    assert info["n_window_groups"] >= 4 * 90_000
    check_rows(ctx, o, "amg full")
    ctx.query(Q_WINDOW, t0=T // 3, t1=T // 2)
    check_rows(ctx, oracle.window(tr, parent, T // 3, T // 2), "amg part")


def test_large_tree_cube_and_outliers(gpu_ctx_factory):
    """The cube of an anchor subtree inside a 50k-context tree (the fused kernel
    reads its column offsets from the global table) and the outlier step on a
    sparse window (site values looked up in the remat rows)."""
    rng = np.random.default_rng(29)
    ctx = gpu_ctx_factory()
    n_ctx = 50_000
    parent = _large_tree(rng, n_ctx)
    # iterations: the anchor subtree {a, its children} entered regularly,
    # other contexts drawn from the whole tree in between
    size = np.ones(n_ctx, np.int64)
    for c in range(n_ctx - 1, 0, -1):
        size[parent[c]] += size[c]
    anchor = int(np.flatnonzero((size >= 4) & (size <= 40))[0])
    kids = np.flatnonzero(parent == anchor).astype(np.uint32)
    ts, cx, off, tend = [], [], [0], []
    for t in range(16):
        now = int(rng.integers(0, 30))
        for it in range(int(rng.integers(5, 12))):
            for c in [anchor, *rng.choice(kids, size=3), *rng.integers(0, n_ctx, size=5)]:
                cx.append(int(c))
                ts.append(now)
                now += int(rng.integers(0, 50))
        off.append(len(ts))
        tend.append(now + 3)
    tr = {"ts": np.array(ts, np.uint64), "ctx": np.array(cx, np.uint32), "off": np.array(off, np.uint64),
          "t_end": np.array(tend, np.uint64), "pid": np.arange(1, 17, dtype=np.uint32)}
    ctx.set_cct(parent)
    ctx.load_aos(to_aos(tr), tr["off"], tr["pid"], tr["t_end"])
    check_cube(ctx, tr, parent, anchor)
    # a whole query: sparse window + cube + outliers over 4 nodes
    T = int(tr["t_end"].max())
    node = np.arange(16) // 4
    ctx.set_nodes(node, 4, 4000 + node // 2, node % 2)
    sites = [anchor, int(kids[0])]
    info = ctx.query(Q_WINDOW | Q_CUBE | Q_STATS | Q_OUTLIERS, t0=T // 4, t1=3 * T // 4, anchor=anchor,
                     sites=sites, top_k=2, z_min=-1e9)
    assert info["window_sparse"] == 1
    o = oracle.window(tr, parent, T // 4, 3 * T // 4)
    check_rows(ctx, o, "full query")
    vals = np.stack([o["incl"][:, s] for s in sites])
    oo = oracle.outliers(vals, node, 4, 2, -1e9)
    out = ctx.outliers(4)
    assert info["worst_site"] == sites[oo["worst"]]
    assert_rel(out["site_ratio"], oo["site_ratio"], 1e-12, "site ratio")
    assert_rel(out["node_mean"], oo["node_mean"], 1e-12, "node mean")
    assert np.array_equal(out["selected"], oo["selected"])

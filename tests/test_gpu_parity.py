"""GPU parity: libpsg.so (through its C ABI) against the CPU oracle
restatement and the reference itself (oracle/_ref), on identical inputs.

Bar (north star): bit-exact for counts, sums, boundaries, cube cells, outlier
ids; 1e-9 relative for the fp64 diagnostics (savings, CV)."""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

import oracle
from paper_2605_03561_b200 import Q_ALL, Q_CLAMP_TEND, Q_CUBE, Q_CUBE64, Q_EXACT_BOUNDS, Q_OUTLIERS, Q_STATS, Q_WINDOW, PsgError, scenarios
from tests.helpers import ROOT, assert_rel, random_cct, random_traces, ref_db, to_aos

pytestmark = pytest.mark.gpu

WINDOW_KEYS = ["count", "sum", "min", "max", "mean", "excl", "incl"]


def check_window(ctx, tr, parent, t0, t1):
    ctx.query(Q_WINDOW, t0=t0, t1=t1)
    g = ctx.window()
    o = oracle.window(tr, parent, t0, t1)
    for k in WINDOW_KEYS:
        assert np.array_equal(g[k], o[k]), f"window {k} differs for [{t0},{t1})"
    gc = ctx.carry()
    for k in ("has", "ts", "ctx"):
        assert np.array_equal(gc[k], o["carry"][k]), f"carry {k}"


def check_cube(ctx, tr, parent, anchor, stats=True):
    """Both HBM cube formats (32-bit cells where every iteration spans < 2^32
    ns, and forced 64-bit cells) and both pass-1 modes (optimistic, verified by
    pass 2, and exact) against the oracle."""
    o = oracle.cube(tr, parent, anchor)
    kept = int((o["iter_counts"] > 0).sum())
    for extra in (0, Q_CUBE64, Q_EXACT_BOUNDS):
        info = ctx.query(Q_CUBE | (Q_STATS if stats else 0) | extra, anchor=anchor)
        if extra == Q_CUBE64 or kept == 0:
            assert info["cube_cell_bytes"] == 8 or kept == 0
        g = ctx.cube()
        for k in ("node_ids", "iter_counts", "block_offset", "incl", "excl", "gap_incl", "gap_excl"):
            assert np.array_equal(g[k], o[k]), f"cube {k} differs (anchor {anchor}, flags {extra})"
        check_stored(ctx, g, parent)
        assert info["n_kept"] == kept
        if stats and kept > 0:
            s = ctx.stats(1.0)
            for j, leaf in enumerate(s["leaves"]):
                npos = int(np.searchsorted(o["node_ids"], leaf))
                want, ok = oracle.node_stats(o, npos)
                # savings = avg_max - avg_mean: a difference of two aggregates, so
                # the 1e-9 bound is relative to the aggregates (identical values
                # make it 0 up to their rounding)
                assert_rel(s["savings"][j][:2], want[:2], 1e-9, f"savings leaf {leaf}")
                assert_rel(s["savings"][j][2:], want[2:4], 1e-9, f"savings leaf {leaf}",
                           atol=1e-9 * abs(want[1]) * max(1, int(info["min_iterations"])))
                assert bool(s["cv_ok"][j]) == ok, f"cv_ok leaf {leaf}"
                if ok:
                    # identical values: exactly 0 from integer sums, rounding noise
                    # from the reference's two-pass fp64 CV (absolute floor 1e-9 %)
                    assert_rel(s["cv"][j], want[4:], 1e-9, f"cv leaf {leaf}", atol=1e-9)
    return g, o


# ---------------------------------------------------------------------------
def test_device_generator_is_byte_identical_to_reference(gpu_ctx_factory):
    ctx = gpu_ctx_factory()
    for cfg in (scenarios.small(seed=52, n_ranks=4, n_iterations=7, jitter=0.1),
                scenarios.iterative(37, 9, n_kernels=5, seed=11, jitter=0.3),
                scenarios.c2(n_ranks=3)):
        d = ref_db(cfg)
        ref = oracle.read_trace_db(d)
        ctx.generate_iterative(cfg)
        g = ctx.traces()
        for k in ("ts", "ctx", "off", "t_end", "pid"):
            assert np.array_equal(g[k], ref[k]), f"generator {k} differs"
        # a rank sub-range is the same bytes as those ranks of the full scenario
        ctx.generate_iterative(cfg, 1, cfg["n_ranks"])
        g2 = ctx.traces()
        a = int(ref["off"][1])
        assert np.array_equal(g2["ts"], ref["ts"][a:]) and np.array_equal(g2["ctx"], ref["ctx"][a:])


def test_trace_db_reader_and_aos_loader_agree(gpu_ctx_factory):
    ctx = gpu_ctx_factory()
    d = ref_db(scenarios.small(seed=3, n_ranks=5, n_iterations=4, jitter=0.2))
    ref = oracle.read_trace_db(d)
    ctx.load_trace_db(d)
    g = ctx.traces()
    for k in ("ts", "ctx", "off", "t_end", "pid"):
        assert np.array_equal(g[k], ref[k])
    meta = oracle.read_meta(d)
    ctx.set_cct(meta["parent"])
    ctx.load_aos(ref["body"], ref["off"], ref["pid"], ref["t_end"])
    g = ctx.traces()
    for k in ("ts", "ctx", "off", "t_end", "pid"):
        assert np.array_equal(g[k], ref[k])
    # subset of pids (gathered path)
    ctx.load_trace_db(d, [4, 2])
    g = ctx.traces()
    assert list(g["pid"]) == [2, 4]


def test_window_matches_reference_composition(gpu_ctx_factory):
    """ingest_traces + dur glue + group_aggregate + rematerialize, straight from oracle/_ref."""
    ctx = gpu_ctx_factory()
    d = ref_db(scenarios.iterative(50, 20, n_kernels=8, seed=5))
    tr = oracle.read_trace_db(d)
    ctx.load_trace_db(d)
    T = int(tr["t_end"].max())
    for t0, t1 in ((T // 4, 3 * T // 4), (0, T), (T // 3, T // 3 + 1), (T + 10, T + 20)):
        ctx.query(Q_WINDOW, t0=t0, t1=t1)
        g = ctx.window()
        r = oracle.ref_window(d, t0, t1)
        row = {int(p): i for i, p in enumerate(tr["pid"])}
        ti = np.array([row[int(p)] for p in r["wa_pid"]], dtype=np.int64)
        ci = r["wa_ctx"].astype(np.int64)
        assert int((g["count"] > 0).sum()) == len(ti)
        assert np.array_equal(g["count"][ti, ci], r["wa_count"])
        assert np.array_equal(g["sum"][ti, ci], r["wa_sum"])
        assert np.array_equal(g["min"][ti, ci], r["wa_min"])
        assert np.array_equal(g["max"][ti, ci], r["wa_max"])
        assert np.array_equal(g["mean"][ti, ci], r["wa_mean"])
        rt = np.array([row[int(p)] for p in r["rm_pid"]], dtype=np.int64)
        assert np.array_equal(g["incl"][rt, r["rm_ctx"]], r["rm_incl"])
        assert np.array_equal(g["excl"][rt, r["rm_ctx"]], r["rm_excl"])
        assert int(((g["incl"] != 0) | (g["excl"] != 0)).sum()) == len(rt)
        c = ctx.carry()
        ct = np.array([row[int(p)] for p in r["carry_pid"]], dtype=np.int64)
        assert np.array_equal(c["has"][ct], r["carry_has"])
        assert np.array_equal(c["ts"][ct], r["carry_ts"])
        assert np.array_equal(c["ctx"][ct], r["carry_ctx"])


def test_window_rows_match_ingest_traces(gpu_ctx_factory):
    ctx = gpu_ctx_factory()
    d = ref_db(scenarios.iterative(30, 10, n_kernels=6, seed=8))
    tr = oracle.read_trace_db(d)
    ctx.load_trace_db(d)
    T = int(tr["t_end"].max())
    for t0, t1 in ((T // 4, 3 * T // 4), (T // 2, T // 2), (0, 1)):
        g = ctx.window_rows(t0, t1)
        r = oracle.ref_window(d, t0, t1, rows=True)
        assert np.array_equal(g["pid"], r["rows_pid"])
        assert np.array_equal(g["ts"], r["rows_ts"])
        assert np.array_equal(g["ctx"], r["rows_ctx"])
        assert np.array_equal(g["carry"]["has"], r["carry_has"])
        assert np.array_equal(g["carry"]["ts"], r["carry_ts"])
    with pytest.raises(PsgError) as e:
        ctx.window_rows(5, 4)
    assert e.value.name == "invalid_argument"


def check_stored(ctx, g, parent):
    """psg_get_cube_stored (the lossless compact copy-out) rebuilds the dense
    cube: incl rows from the padded blocks, excl = incl for leaves and the
    compact internal-node rows for the rest."""
    st = ctx.cube_stored()
    nn, ic = len(g["node_ids"]), g["iter_counts"]
    ids = set(int(x) for x in g["node_ids"])
    internal = [j for j, c in enumerate(g["node_ids"])
                if any(int(parent[x]) == int(c) for x in ids if x != c and parent[x] != 0xFFFFFFFF)]
    rows = []
    for t in np.flatnonzero(ic):
        o = int(st["stored_off"][t])
        rows.append(st["incl"][o:o + int(ic[t]) * st["row_stride"]].reshape(-1, st["row_stride"])[:, :nn])
    incl = np.concatenate(rows).astype(np.int64) if rows else np.zeros((0, nn), np.int64)
    assert np.array_equal(incl.ravel(), g["incl"]), "stored incl"
    excl = incl.copy()
    if internal and len(incl):
        excl[:, internal] = st["xint"].reshape(len(incl), len(internal))
    assert np.array_equal(excl.ravel(), g["excl"]), "stored excl"
    # the asynchronous copy-out lands the same bytes
    a = ctx.cube_stored(np.zeros_like(st["incl"]), np.zeros_like(st["xint"]), wait=False)
    ctx.wait_copies()
    for k in ("incl", "xint", "stored_off"):
        assert np.array_equal(a[k], st[k]), f"async stored {k}"


def test_cube_matches_build_tri_model(gpu_ctx_factory):
    ctx = gpu_ctx_factory()
    for cfg, anchor in ((scenarios.small(seed=54, n_ranks=5, n_iterations=6, jitter=0.3), 1),
                        (scenarios.iterative(40, 30, n_kernels=12, seed=9, spread="gamess"), 1),
                        (scenarios.small(seed=55, n_ranks=2, n_iterations=3), 0)):
        d = ref_db(cfg)
        ctx.load_trace_db(d)
        ctx.query(Q_CUBE | Q_STATS, anchor=anchor)
        g = ctx.cube()
        r = oracle.ref_trimodel(d, anchor)
        for k in ("node_ids", "incl", "excl", "gap_incl", "gap_excl", "block_offset"):
            assert np.array_equal(g[k], r[k]), k
        assert np.array_equal(g["iter_counts"][g["iter_counts"] > 0], r["iter_counts"])
        s = ctx.stats(float(r["savings_summary"][2]))
        assert np.array_equal(s["leaves"], r["leaves"])
        assert_rel(s["savings"].ravel(), r["savings"], 1e-9, "savings")
        assert_rel(s["summary"], r["savings_summary"], 1e-9, "summary")
        cv_ok = r["cv_ok"].astype(bool)
        assert np.array_equal(s["cv_ok"].astype(bool), cv_ok)
        assert_rel(s["cv"][cv_ok].ravel(), r["cv"].reshape(-1, 2)[cv_ok].ravel(), 1e-9, "cv")


@pytest.mark.parametrize("seed", range(6))
def test_random_traces_property(gpu_ctx_factory, seed):
    """Random CCTs / traces with equal timestamps, repeated contexts inside a
    warp, empty traces and t_end == last ts: GPU == oracle bit for bit."""
    rng = np.random.default_rng(seed)
    ctx = gpu_ctx_factory()
    n_ctx = int(rng.integers(3, 40))
    parent = random_cct(rng, n_ctx)
    tr = random_traces(rng, int(rng.integers(1, 60)), n_ctx, int(rng.integers(1, 900)),
                       ctx_pool=int(rng.integers(2, n_ctx + 1)), dup_prob=float(rng.random()) * 0.6)
    ctx.set_cct(parent)
    ctx.load_aos(to_aos(tr), tr["off"], tr["pid"], tr["t_end"])
    T = int(tr["t_end"].max()) if len(tr["t_end"]) else 10
    for t0, t1 in ((0, T + 1), (T // 3, 2 * T // 3), (T // 2, T // 2), (T // 5, T // 5 + 7)):
        check_window(ctx, tr, parent, t0, t1)
    for anchor in sorted({0, 1, int(rng.integers(0, n_ctx)), n_ctx - 1}):
        check_cube(ctx, tr, parent, anchor)


def test_long_traces_cross_many_chunks(gpu_ctx_factory):
    rng = np.random.default_rng(99)
    ctx = gpu_ctx_factory()
    parent = np.array([0xFFFFFFFF, 0, 1, 1, 2, 0], np.uint32)
    tr = random_traces(rng, 9, 6, 20000, ts_step=30, dup_prob=0.2)
    ctx.set_cct(parent)
    ctx.load_aos(to_aos(tr), tr["off"], tr["pid"], tr["t_end"])
    T = int(tr["t_end"].max())
    check_window(ctx, tr, parent, T // 7, T // 2)
    for anchor in (1, 2, 3):
        check_cube(ctx, tr, parent, anchor)


def test_format_errors_fail_loudly(gpu_ctx_factory):
    ctx = gpu_ctx_factory()
    parent = np.array([0xFFFFFFFF, 0, 1], np.uint32)
    ctx.set_cct(parent)
    tr = {"ts": np.array([5, 3], np.uint64), "ctx": np.array([1, 2], np.uint32),
          "off": np.array([0, 2], np.uint64), "t_end": np.array([9], np.uint64),
          "pid": np.array([1], np.uint32)}
    with pytest.raises(PsgError) as e:
        ctx.load_aos(to_aos(tr), tr["off"], tr["pid"], tr["t_end"])
    assert e.value.name == "format_error"
    tr["ts"] = np.array([3, 5], np.uint64)
    tr["ctx"] = np.array([1, 7], np.uint32)  # dangling ctx
    with pytest.raises(PsgError):
        ctx.load_aos(to_aos(tr), tr["off"], tr["pid"], tr["t_end"])
    with pytest.raises(PsgError) as e:
        ctx.set_cct(np.array([0xFFFFFFFF, 2, 0], np.uint32))
    assert e.value.name == "format_error"


def test_c1_window_at_full_size(gpu_ctx_factory):
    """BASELINE configs[0] at full size: 1,000 x 10,050 events, window [T/4, 3T/4).
    The reference composition runs here too (a few seconds)."""
    ctx = gpu_ctx_factory()
    cfg = scenarios.c1()
    d = ref_db(cfg)
    ctx.generate_iterative(cfg)
    tr = oracle.read_trace_db(d)
    g = ctx.traces()
    assert np.array_equal(g["ts"], tr["ts"]) and np.array_equal(g["ctx"], tr["ctx"])
    T = int(tr["t_end"].max())
    check_window(ctx, tr, oracle.read_meta(d)["parent"], T // 4, 3 * T // 4)


def test_congestion_outliers_match_reference(gpu_ctx_factory):
    """C4 shape (aurora_like_config): the z-score / top-k selection over node
    means equals the reference congestion_report outlier group (DBSCAN) and
    the generator truth; racks equal the injected 22."""
    ctx = gpu_ctx_factory()
    cfg = scenarios.aurora(ranks_per_node=10, seed=2025)
    d = ref_db(cfg)
    truth = json.load(open(f"{d}/truth.json"))
    ctx.load_trace_db(d)
    meta = oracle.read_meta(d)
    sites = truth["callsite_ctx"]
    whole = dict(t0=0, t1=2**64 - 1, sites=sites)
    ctx.query(Q_WINDOW | Q_OUTLIERS | Q_CLAMP_TEND, top_k=0, z_min=1.0, **whole)
    info = ctx.info
    rep = json.loads(oracle.ref_congestion_report(d))
    want_ratio = [s["balance_ratio"] for s in rep["callsites"]]
    assert [s["ctx_id"] for s in rep["callsites"]] == sites
    assert info["worst_site"] == rep["worst"]["ctx_id"] == truth["congested_ctx"]
    assert abs(info["worst_ratio"] - rep["worst"]["balance_ratio"]) <= 1e-9 * rep["worst"]["balance_ratio"]
    hosts = sorted({h for (_, r, h) in meta["profiles"] if r >= 0})
    out = ctx.outliers(len(hosts))
    assert_rel(out["site_ratio"], want_ratio, 1e-9, "balance ratios")
    got = sorted(hosts[i] for i in out["selected"])
    assert got == sorted(rep["outlier_group"]["hostnames"]) == sorted(truth["outlier_hostnames"])
    racks = [int(r[0]) for r in out["racks"]]
    assert racks == [r["rack"] for r in rep["topology"]["racks"]] == truth["outlier_rack_ids"]
    assert [int(r[1]) for r in out["racks"]] == [r["nodes"] for r in rep["topology"]["racks"]]
    # top-k with k = 202 gives the same set
    ctx.query(Q_WINDOW | Q_OUTLIERS | Q_CLAMP_TEND, top_k=202, **whole)
    out2 = ctx.outliers(len(hosts))
    assert sorted(hosts[i] for i in out2["selected"]) == got


def test_full_query_all_parts(gpu_ctx_factory):
    ctx = gpu_ctx_factory()
    cfg = scenarios.iterative(64, 12, n_kernels=10, seed=21)
    ctx.generate_iterative(cfg)
    tr = ctx.traces()
    parent = np.array([0xFFFFFFFF, 0] + [1] * 10 + [0], np.uint32)
    node = np.arange(64) // 8
    ctx.set_nodes(node, 8, 4000 + node // 4, node % 4)
    T = int(tr["t_end"].max())
    info = ctx.query(Q_ALL, t0=T // 4, t1=3 * T // 4, anchor=1, sites=[2, 3, 4], top_k=3, z_min=-1e9)
    assert info["n_kept"] == 64 and info["min_iterations"] == 12
    w = ctx.window()
    o = oracle.window(tr, parent, T // 4, 3 * T // 4)
    for k in WINDOW_KEYS:
        assert np.array_equal(w[k], o[k])
    g = ctx.cube()
    oc = oracle.cube(tr, parent, 1)
    assert np.array_equal(g["incl"], oc["incl"])
    vals = np.stack([o["incl"][:, s] for s in (2, 3, 4)])
    oo = oracle.outliers(vals, node, 8, 3, -1e9)
    out = ctx.outliers(8)
    assert info["worst_site"] == [2, 3, 4][oo["worst"]]
    assert_rel(out["site_ratio"], oo["site_ratio"], 1e-12, "site ratio")
    assert_rel(out["node_mean"], oo["node_mean"], 1e-12, "node mean")
    assert np.array_equal(out["selected"], oo["selected"])


@pytest.mark.parametrize("seed", range(3))
def test_wide_durations(gpu_ctx_factory, seed):
    """Segments, iterations and block steps spanning >= 2^31 / 2^32 ns take the
    64-bit paths (carried shared adds, big min/max, 128-bit squares): still
    bit-exact against the oracle."""
    rng = np.random.default_rng(500 + seed)
    ctx = gpu_ctx_factory()
    n_ctx = int(rng.integers(3, 12))
    parent = random_cct(rng, n_ctx)
    tr = random_traces(rng, int(rng.integers(2, 20)), n_ctx, int(rng.integers(50, 700)),
                       ts_step=2**34, dup_prob=0.3)
    ctx.set_cct(parent)
    ctx.load_aos(to_aos(tr), tr["off"], tr["pid"], tr["t_end"])
    T = int(tr["t_end"].max())
    for t0, t1 in ((0, T + 1), (T // 3, 2 * T // 3), (T // 5, T // 5 + 2**33)):
        check_window(ctx, tr, parent, t0, t1)
    for anchor in sorted({0, 1, int(rng.integers(0, n_ctx))}):
        check_cube(ctx, tr, parent, anchor)


@pytest.mark.parametrize("long_span", [3 * 2**31, 2**30])
def test_narrow_and_wide_iterations_mixed(gpu_ctx_factory, long_span):
    """One trace whose iterations alternate between short (< 2^30 ns) and
    long spans: chunks switch between the 32-bit and the 64-bit shared-memory
    cube paths inside one trace.  Long iterations > 2^32 ns force 64-bit HBM
    cells; 2^31 ns ones keep 32-bit HBM cells with 64-bit shared rows."""
    parent = np.array([0xFFFFFFFF, 0, 1, 1, 0], np.uint32)
    ts, cx = [], []
    t = 1000
    for it in range(40):
        long_it = (it // 3) % 2 == 1
        ts.append(t); cx.append(1)
        for k in (2, 3):
            ts.append(t); cx.append(k)
            t += (long_span if long_it else 10_000 + 37 * it) + k
        ts.append(t); cx.append(4)
        t += 5
        ts.append(t); cx.append(0)
        t += 3
    tr = {"ts": np.array(ts, np.uint64), "ctx": np.array(cx, np.uint32),
          "off": np.array([0, len(ts)], np.uint64), "t_end": np.array([t + 7], np.uint64),
          "pid": np.array([1], np.uint32)}
    ctx = gpu_ctx_factory()
    ctx.set_cct(parent)
    ctx.load_aos(to_aos(tr), tr["off"], tr["pid"], tr["t_end"])
    for anchor in (1, 0):
        check_cube(ctx, tr, parent, anchor, stats=False)
    check_window(ctx, tr, parent, 0, t + 8)


def test_auto_anchor_on_device_matches_reference(gpu_ctx_factory):
    """PSG_ANCHOR_AUTO runs suggest_anchor on the device over the trace with the
    smallest profile id; the reference's choice (golden), then the same cube."""
    from paper_2605_03561_b200 import ANCHOR_AUTO
    from tests.test_oracle import load
    ctx = gpu_ctx_factory()
    z = load("anchor_cases")
    for i in range(int(z["n_cases"][0])):
        tr = {k: z[f"case{i}_{k}"] for k in ("ts", "ctx", "off", "t_end", "pid")}
        want = int(z[f"case{i}_anchor"][0])
        ctx.set_cct(z["parent"])
        ctx.load_aos(to_aos(tr), tr["off"], tr["pid"], tr["t_end"])
        if want == 0xFFFFFFFF:
            with pytest.raises(PsgError) as e:
                ctx.query(Q_CUBE, anchor=ANCHOR_AUTO)
            assert e.value.name == "no_periodicity"
            continue
        info = ctx.query(Q_CUBE, anchor=ANCHOR_AUTO)
        assert info["anchor"] == want, i
        assert np.array_equal(ctx.cube()["incl"], oracle.cube(tr, z["parent"], want)["incl"])
    for name in ("small_iter", "gamess_like"):
        g = load(name)
        tr = {k: g[k] for k in ("ts", "ctx", "off", "t_end", "pid")}
        ctx.set_cct(g["parent"])
        ctx.load_aos(to_aos(tr), tr["off"], tr["pid"], tr["t_end"])
        info = ctx.query(Q_CUBE | Q_STATS, anchor=ANCHOR_AUTO)
        assert info["anchor"] == int(g["auto_anchor"][0])


def test_trace_db_ingest_multi_buffer(gpu_ctx_factory, tmp_path):
    """psg_load_trace_db through the pread -> pinned ring -> HBM pipeline over
    several 4 Mi-event buffers, and the page-cache-free gathered path for a
    subset: the loaded events equal the ones written."""
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from load_bench import write_db
    ctx = gpu_ctx_factory()
    ctx.generate_iterative(scenarios.device_scenario(260, 746, seed=4))  # 13.0 M events
    want = ctx.traces()
    parent = np.array([0xFFFFFFFF, 0] + [1] * 64 + [0], np.uint32)
    d = str(tmp_path / "db")
    write_db(ctx, d, parent)
    ctx.load_trace_db(d)
    got = ctx.traces()
    for k in ("ts", "ctx", "off", "t_end", "pid"):
        assert np.array_equal(got[k], want[k]), k
    sub = [int(want["pid"][i]) for i in (3, 100, 257)]
    ctx.load_trace_db(d, sub)
    g2 = ctx.traces()
    assert list(g2["pid"]) == sub
    a = int(want["off"][100])
    assert np.array_equal(g2["ts"][int(g2["off"][1]):int(g2["off"][2])],
                          want["ts"][a:a + int(g2["off"][2] - g2["off"][1])])


def test_candidates_sharing_a_timestamp(gpu_ctx_factory):
    """The optimistic pass 1 takes every subtree entry as a boundary; an entry
    on the same timestamp as the previous one (itermodel.cpp:121-130 drops
    it) must be caught by pass 2 and re-run exactly -- on the first query and
    on later ones (which start exact)."""
    parent = np.array([0xFFFFFFFF, 0, 1, 0], np.uint32)
    ev = [(10, 1), (20, 2), (30, 3), (30, 1), (30, 3), (30, 1), (40, 2), (50, 3), (60, 1), (70, 2)]
    tr = {"ts": np.array([t for t, _ in ev] * 3, np.uint64),
          "ctx": np.array([c for _, c in ev] * 3, np.uint32),
          "off": np.array([0, 10, 20, 30], np.uint64), "t_end": np.array([80, 80, 80], np.uint64),
          "pid": np.array([1, 2, 3], np.uint32)}
    # second and third traces: shifted copies without the duplicate entry
    tr["ts"][10:20] += 1000
    tr["ts"][20:30] += 2000
    tr["ctx"][24] = 2
    tr["t_end"][1:] += np.array([1000, 2000], np.uint64)
    ctx = gpu_ctx_factory()
    ctx.set_cct(parent)
    ctx.load_aos(to_aos(tr), tr["off"], tr["pid"], tr["t_end"])
    for _ in range(2):
        g, o = check_cube(ctx, tr, parent, 1)
    assert list(o["iter_counts"][:1]) == [3]


@pytest.mark.parametrize("n_kernels", [1, 2, 3, 4, 33, 36])
def test_flush_tail_columns(gpu_ctx_factory, n_kernels):
    """Leaf counts whose last group of 32 columns holds 1..4 leaves: the fast
    flush takes those columns one cell per lane (row sums, within-rank sums)
    -- cube, savings and CVs still equal the reference."""
    cfg = scenarios.iterative(6, 21, n_kernels=n_kernels, seed=60 + n_kernels, jitter=0.2)
    d = ref_db(cfg)
    tr = oracle.read_trace_db(d)
    parent = oracle.read_meta(d)["parent"]
    ctx = gpu_ctx_factory()
    ctx.set_cct(parent)
    ctx.load_aos(to_aos(tr), tr["off"], tr["pid"], tr["t_end"])
    check_cube(ctx, tr, parent, 1)


def test_flush_tail_columns_with_large_cells(gpu_ctx_factory):
    """Tail leaves with cells >= 2^30 ns (and < 2^32: 32-bit cells): the tail's
    squares are summed in 128 bits."""
    parent = np.array([0xFFFFFFFF, 0, 1, 1, 0], np.uint32)
    ts, cx = [], []
    t = 1000
    for it in range(26):
        ts.append(t); cx.append(1)
        for k in (2, 3):
            ts.append(t); cx.append(k)
            t += (2**30 + 12345 * it + k) if (it + k) % 3 else 777 + it
        ts.append(t); cx.append(4)
        t += 5
        ts.append(t); cx.append(0)
        t += 3
    tr = {"ts": np.array(ts, np.uint64), "ctx": np.array(cx, np.uint32),
          "off": np.array([0, len(ts)], np.uint64), "t_end": np.array([t + 7], np.uint64),
          "pid": np.array([1], np.uint32)}
    ctx = gpu_ctx_factory()
    ctx.set_cct(parent)
    ctx.load_aos(to_aos(tr), tr["off"], tr["pid"], tr["t_end"])
    check_cube(ctx, tr, parent, 1)


@pytest.mark.parametrize("n_ctx", [127, 128, 129, 256])
def test_pass1_membership_at_ctx8_edges(gpu_ctx_factory, n_ctx):
    """Pass 1 on the 1-byte preorder mirror at the edges of its two subtree
    tests: the 3-op SWAR test (every preorder byte < 128: n_ctx <= 128, incl.
    the root's subtree [0, 128) whose upper bound has no headroom) and the
    SIMD-compare test above it (129..256 contexts); anchors at the first and
    last preorder positions and a random one.  GPU == oracle bit for bit."""
    rng = np.random.default_rng(1000 + n_ctx)
    ctx = gpu_ctx_factory()
    parent = random_cct(rng, n_ctx)
    tr = random_traces(rng, 12, n_ctx, 3000, ctx_pool=n_ctx, dup_prob=0.3)
    ctx.set_cct(parent)
    ctx.load_aos(to_aos(tr), tr["off"], tr["pid"], tr["t_end"])
    for anchor in sorted({0, 1, n_ctx - 1, int(rng.integers(0, n_ctx))}):
        check_cube(ctx, tr, parent, anchor, stats=False)


def test_prefetched_loads_equal_plain_loads(gpu_ctx_factory):
    """psg_prefetch_aos (the e2e pipelining hint): a pinned load whose first two
    768 MB staging chunks were copied while a query ran equals the plain load
    (a third chunk follows the prefetched two: 150 M events); a prefetch of
    another length, or one followed by another staging user (export), is
    dropped and the load is still exact.  Checked on the loaded events and on
    a full query's window and cube."""
    import torch
    ctx = gpu_ctx_factory()
    ctx.generate_iterative(scenarios.device_scenario(3000, 746, seed=6))  # 149.9 M events
    n_ev = ctx.shard()["n_events"]
    assert n_ev > 2 * (64 << 20)
    idx = ctx.index()
    host = torch.empty(n_ev * 12, dtype=torch.uint8, pin_memory=True)
    ctx.export_aos(host.data_ptr())
    parent = np.array([0xFFFFFFFF, 0] + [1] * 64 + [0], np.uint32)
    ctx.set_cct(parent)
    T = int(ctx.shard()["t_max"])

    def run():
        ctx.query(Q_WINDOW | Q_CUBE | Q_STATS, t0=T // 4, t1=3 * T // 4, anchor=1)
        return ctx.window(), ctx.cube()

    ctx.load_aos(host.data_ptr(), idx["off"], idx["pid"], idx["t_end"])
    want_ev = ctx.traces()
    want_w, want_c = run()
    # prefetched (query in between), then loaded
    ctx.prefetch_aos(host.data_ptr(), n_ev)
    run()
    ctx.load_aos(host.data_ptr(), idx["off"], idx["pid"], idx["t_end"])
    got = ctx.traces()
    for k in ("ts", "ctx", "off"):
        assert np.array_equal(got[k], want_ev[k]), k
    w, c = run()
    for k in WINDOW_KEYS:
        assert np.array_equal(w[k], want_w[k]), k
    for k in ("iter_counts", "incl", "excl", "gap_incl"):
        assert np.array_equal(c[k], want_c[k]), k
    # a prefetch that does not match the load, and one another staging user drops
    ctx.prefetch_aos(host.data_ptr(), n_ev - 5)
    ctx.load_aos(host.data_ptr(), idx["off"], idx["pid"], idx["t_end"])
    assert np.array_equal(ctx.traces()["ts"], want_ev["ts"])
    ctx.prefetch_aos(host.data_ptr(), n_ev)
    out = torch.empty(n_ev * 12, dtype=torch.uint8, pin_memory=True)
    ctx.export_aos(out.data_ptr())
    assert torch.equal(out, host)
    ctx.load_aos(host.data_ptr(), idx["off"], idx["pid"], idx["t_end"])
    got = ctx.traces()
    assert np.array_equal(got["ts"], want_ev["ts"]) and np.array_equal(got["ctx"], want_ev["ctx"])

"""GPU parity at the benchmarked sizes (BASELINE.json configs[1], [2], [3]).

configs[1] (100,000 traces x 49,982 events, 5.0e9 events, the bench.py
workload): the full query runs on the device over all traces, exactly as
bench.py runs it; the traces of ranks 0..399 and 99,600..99,999 are exported
from HBM (psg_export_aos_range), written as a trace.db by the reference's own
writer, and the UNMODIFIED reference (oracle/_ref) computes ingest_traces +
group_aggregate + rematerialize over the same window and build_tri_model with
anchor 1 on them.  Window rows, carry-ins, iteration counts, cube cells and gap
rows must be bit-identical.  The second range sits above 2^32 cube cells
(offset ~4.9e9), so the 64-bit cube addressing is exercised.  Size-independent
properties cover all 100,000 traces (window counts against the independent
window-bounds kernel, every trace's iteration count).

configs[2] (C3: 8,192 GAMESS-like ranks x 500 iterations x 64 kernels, written
by the reference generator): the whole cube, gap rows, block offsets and the
diagnostics against the reference (tools/c3_check.py, now in the suite).

configs[3] (C4: aurora-like 1,000 nodes x 100 ranks): the z >= 1 and top-202
outlier sets equal the reference congestion_report's DBSCAN group and the
generator truth, on both the trace path and the profile-record path.
"""
from __future__ import annotations

import json
import os
import tempfile

import numpy as np
import pytest

import oracle
from paper_2605_03561_b200 import Q_ALL, Q_CLAMP_TEND, Q_CUBE, Q_OUTLIERS, Q_STATS, Q_WINDOW, Context, scenarios
from tests.helpers import assert_rel, ref_db

pytestmark = pytest.mark.gpu

N = 100_000
ITERS = 746
RANGES = [(0, 400), (N - 400, N)]
_REF: dict = {}


@pytest.fixture(scope="module")
def c2():
    """configs[1] on the device, set up like bench.py."""
    ctx = Context(0)
    ctx.generate_iterative(scenarios.c2_device(N))
    sh = ctx.shard()
    node_of = (np.arange(N) // 100).astype(np.uint32)
    n_nodes = N // 100
    node = np.arange(n_nodes)
    ctx.set_nodes(node_of, n_nodes, 4000 + node // 32, (node // 8) % 4)
    T = int(sh["t_max"])
    q = dict(flags=Q_ALL, t0=T // 4, t1=3 * T // 4, anchor=1, sites=list(range(2, 66)), top_k=32)
    yield ctx, T, q
    ctx.close()


def _reference_for_range(ctx, lo, hi, T):
    """oracle/_ref on the exported traces [lo, hi) (cached across CTA shapes)."""
    key = (lo, hi)
    if key in _REF:
        return _REF[key]
    body = ctx.export_aos_range(lo, hi).reshape(-1, 12)
    idx = ctx.index()
    off = idx["off"][lo:hi + 1] - idx["off"][lo]
    tr = {"ts": body[:, :8].copy().view(np.uint64).ravel(), "ctx": body[:, 8:].copy().view(np.uint32).ravel(),
          "off": off, "t_end": idx["t_end"][lo:hi], "pid": idx["pid"][lo:hi]}
    parent = np.array([0xFFFFFFFF, 0] + [1] * 64 + [0], np.uint32)
    base = "/dev/shm" if os.path.isdir("/dev/shm") else None
    with tempfile.TemporaryDirectory(dir=base) as d:
        oracle.ref_write_traces(tr, parent, d)
        jobs = int(oracle.ref().refh_default_jobs())
        r = {"window": oracle.ref_window(d, T // 4, 3 * T // 4, jobs=jobs),
             "cube": oracle.ref_trimodel(d, 1, jobs=jobs), "pid": tr["pid"]}
    _REF[key] = r
    return r


def test_configs1_full_query_equals_reference_on_both_rank_ends(c2):
    ctx, T, q = c2
    info = ctx.query(**q)
    assert info["n_kept"] == N and info["min_iterations"] == ITERS
    w = ctx.window()
    carry = ctx.carry()
    ic = ctx.cube(with_cells=False)["iter_counts"]
    # size-independent properties over all traces: every trace has 746
    # iterations; the fused kernel's per-trace window row counts equal the
    # window-bounds kernel's (psg_window_rows' binary searches)
    assert (ic == ITERS).all()
    for lo, hi in RANGES:
        r = _reference_for_range(ctx, lo, hi, T)
        rw, rc = r["window"], r["cube"]
        row = {int(p): i for i, p in enumerate(r["pid"])}
        # window: group_aggregate rows + rematerialize + carry-ins
        ti = lo + np.array([row[int(p)] for p in rw["wa_pid"]], dtype=np.int64)
        ci = rw["wa_ctx"].astype(np.int64)
        assert int((w["count"][lo:hi] > 0).sum()) == len(ti)
        for k in ("count", "sum", "min", "max", "mean"):
            assert np.array_equal(w[k][ti, ci], rw["wa_" + k]), (lo, k)
        rt = lo + np.array([row[int(p)] for p in rw["rm_pid"]], dtype=np.int64)
        assert np.array_equal(w["incl"][rt, rw["rm_ctx"]], rw["rm_incl"])
        assert np.array_equal(w["excl"][rt, rw["rm_ctx"]], rw["rm_excl"])
        ct = lo + np.array([row[int(p)] for p in rw["carry_pid"]], dtype=np.int64)
        for k in ("has", "ts", "ctx"):
            assert np.array_equal(carry[k][ct], rw["carry_" + k]), (lo, k)
        # cube: the kept traces of the range, dense int64 (device-widened)
        g = ctx.cube_range(lo, hi)
        assert np.array_equal(ic[lo:hi][ic[lo:hi] > 0], rc["iter_counts"])
        for k in ("incl", "excl", "gap_incl", "gap_excl"):
            assert np.array_equal(g[k], rc[k]), (lo, k)
    # the second range's blocks start above 2^32 cells
    assert int(ic[:RANGES[1][0]].astype(np.uint64).sum()) * info["n_nodes"] > 2**32


def test_configs1_window_rows_agree_across_kernels(c2):
    """Σ window counts (k_trace_query's fused filter) == the rows of
    ingest_traces' window (k_window_bounds' binary searches): two independent
    kernels over all 5e9 events; and the carry-ins of both agree."""
    ctx, T, q = c2
    ctx.query(Q_WINDOW, t0=q["t0"], t1=q["t1"])
    total = int(ctx.window()["count"].sum(dtype=np.uint64))
    c1 = ctx.carry()
    assert total == ctx.window_row_count(q["t0"], q["t1"])
    c2_ = ctx.carry()
    for k in ("has", "ts", "ctx"):
        assert np.array_equal(c1[k], c2_[k]), k


# ---------------------------------------------------------------------------
_C3: dict = {}


def _c3_reference():
    if not _C3:
        d = ref_db(scenarios.c3())
        jobs = int(oracle.ref().refh_default_jobs())
        _C3["d"] = d
        _C3["ref"] = oracle.ref_trimodel(d, 1, jobs=jobs, total_time=100.0)
    return _C3["d"], _C3["ref"]


def test_configs2_c3_full_size_equals_build_tri_model(gpu_ctx_factory):
    d, ref = _c3_reference()
    ctx = gpu_ctx_factory()
    ctx.load_trace_db(d)
    ctx.query(Q_CUBE | Q_STATS, anchor=1)
    g = ctx.cube()
    for k in ("node_ids", "incl", "excl", "gap_incl", "gap_excl", "block_offset"):
        assert np.array_equal(g[k], ref[k]), k
    assert np.array_equal(g["iter_counts"][g["iter_counts"] > 0], ref["iter_counts"])
    s = ctx.stats(float(ref["savings_summary"][2]))
    assert np.array_equal(s["leaves"], ref["leaves"])
    assert_rel(s["savings"].ravel(), ref["savings"], 1e-9, "savings")
    assert_rel(s["summary"], ref["savings_summary"], 1e-9, "summary")
    cv_ok = ref["cv_ok"].astype(bool)
    assert np.array_equal(s["cv_ok"].astype(bool), cv_ok)
    assert_rel(s["cv"][cv_ok].ravel(), ref["cv"].reshape(-1, 2)[cv_ok].ravel(), 1e-9, "cv")


# ---------------------------------------------------------------------------
_C4: dict = {}


def _c4():
    if not _C4:
        cfg = scenarios.aurora(ranks_per_node=100, seed=42)
        d = ref_db(cfg)
        _C4.update(d=d, truth=json.load(open(f"{d}/truth.json")), meta=oracle.read_meta(d),
                   rep=json.loads(oracle.ref_congestion_report(d)))
    return _C4


def _check_c4_outliers(ctx, hosts, c):
    rep, truth = c["rep"], c["truth"]
    info = ctx.info
    assert info["worst_site"] == rep["worst"]["ctx_id"] == truth["congested_ctx"]
    out = ctx.outliers(len(hosts))
    assert_rel(out["site_ratio"], [s["balance_ratio"] for s in rep["callsites"]], 1e-9, "balance ratios")
    got = sorted(hosts[i] for i in out["selected"])
    assert got == sorted(rep["outlier_group"]["hostnames"]) == sorted(truth["outlier_hostnames"])
    assert len(got) == 202
    assert [int(r[0]) for r in out["racks"]] == [r["rack"] for r in rep["topology"]["racks"]]
    assert [int(r[1]) for r in out["racks"]] == [r["nodes"] for r in rep["topology"]["racks"]]
    rows = ctx.topology()
    for e in rep["topology"]["racks"]:
        mine = rows[rows[:, 0] == e["rack"]]
        assert mine[:, 1].tolist() == e["chassis"]
        assert mine[mine[:, 3] == 1, 1].tolist() == e["full_chassis"]
    return got


def test_configs3_c4_full_size_outliers_trace_path(gpu_ctx_factory):
    c = _c4()
    ctx = gpu_ctx_factory()
    ctx.load_trace_db(c["d"])
    hosts = sorted({h for (_, r, h) in c["meta"]["profiles"] if r >= 0})
    whole = dict(t0=0, t1=2**64 - 1, sites=c["truth"]["callsite_ctx"])
    ctx.query(Q_WINDOW | Q_OUTLIERS | Q_CLAMP_TEND, top_k=0, z_min=1.0, **whole)
    got = _check_c4_outliers(ctx, hosts, c)
    ctx.query(Q_WINDOW | Q_OUTLIERS | Q_CLAMP_TEND, top_k=202, **whole)
    assert sorted(hosts[i] for i in ctx.outliers(len(hosts))["selected"]) == got


def test_configs3_c4_full_size_outliers_profile_path(gpu_ctx_factory):
    c = _c4()
    ctx = gpu_ctx_factory()
    ctx.load_profile_db(c["d"])
    metric = next(m for (m, sc, n) in c["meta"]["metrics"] if n == "cputime" and sc == 1)
    hosts = sorted({h for (_, r, h) in c["meta"]["profiles"] if r >= 0})
    ctx.profile_outliers(metric, c["truth"]["callsite_ctx"], top_k=0, z_min=1.0)
    _check_c4_outliers(ctx, hosts, c)

"""CPU suite: pins the oracle (oracle/psg_oracle.c, the CPU restatement) to the
reference's own outputs — golden vectors written by the UNMODIFIED reference
(tests/golden/make_golden.py) and the known-answer tests of the reference's
test suite — and checks the C-ABI library's exported surface.  No GPU."""
from __future__ import annotations

import json
import os
import re

import numpy as np
import pytest

import oracle
from tests.helpers import GOLDEN, ROOT, assert_rel

FIXTURES = ["small_iter", "gamess_like", "random_0", "random_1", "random_2", "random_3"]


def load(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def traces(g: dict) -> dict:
    return {k: g[k] for k in ("ts", "ctx", "off", "t_end", "pid")}


def densify_window(g: dict, i: int, n: int, n_ctx: int) -> dict:
    """Sparse reference rows (group_aggregate / rematerialize) -> dense [trace][ctx]."""
    row = {int(p): t for t, p in enumerate(g["pid"])}
    out = {k: np.zeros((n, n_ctx), dt) for k, dt in [
        ("count", np.uint64), ("sum", np.int64), ("min", np.int64), ("max", np.int64),
        ("mean", np.float64), ("excl", np.int64), ("incl", np.int64)]}
    ti = np.array([row[int(p)] for p in g[f"w{i}_wa_pid"]], np.int64)
    ci = g[f"w{i}_wa_ctx"].astype(np.int64)
    for k in ("count", "sum", "min", "max", "mean"):
        out[k][ti, ci] = g[f"w{i}_wa_{k}"]
    rt = np.array([row[int(p)] for p in g[f"w{i}_rm_pid"]], np.int64)
    out["incl"][rt, g[f"w{i}_rm_ctx"].astype(np.int64)] = g[f"w{i}_rm_incl"]
    out["excl"][rt, g[f"w{i}_rm_ctx"].astype(np.int64)] = g[f"w{i}_rm_excl"]
    ct = np.array([row[int(p)] for p in g[f"w{i}_carry_pid"]], np.int64)
    carry = {"has": np.zeros(n, np.uint8), "ts": np.zeros(n, np.uint64), "ctx": np.zeros(n, np.uint32)}
    carry["has"][ct] = g[f"w{i}_carry_has"]
    carry["ts"][ct] = g[f"w{i}_carry_ts"]
    carry["ctx"][ct] = g[f"w{i}_carry_ctx"]
    out["carry"] = carry
    return out


# ---- known-answer tests from the reference's suite ---------------------------

def test_kat_single_segment():
    """test_itermodel.cpp:77-85: {100, leaf} over [100,105) -> leaf (5,5), mid (5,0), root (5,0)."""
    g = load("kat_single_segment")
    ref = {int(c): (int(i), int(e)) for c, i, e in zip(g["w0_rm_ctx"], g["w0_rm_incl"], g["w0_rm_excl"])}
    assert ref == {2: (5, 5), 1: (5, 0), 0: (5, 0)}
    o = oracle.window(traces(g), g["parent"], 100, 105)
    assert o["excl"][0].tolist() == [0, 0, 5, 0]
    assert o["incl"][0].tolist() == [5, 5, 5, 0]
    assert o["count"][0].tolist() == [0, 0, 1, 0] and o["sum"][0, 2] == 5


def savings_fixture_cube():
    """acceptance.cpp:77-104: 2 traces x 11 iterations x 6 kernels with
    (mean, max) pairs; trace 0 holds 2*mean-max, trace 1 holds max."""
    pairs = [(2.963, 4.650), (2.483, 2.599), (0.734, 0.945), (0.483, 0.958), (0.239, 0.300),
             (0.007, 0.010)]
    nn = len(pairs)
    incl = np.zeros(2 * 11 * nn, np.int64)
    for k, (mean, mx) in enumerate(pairs):
        max_ns = int(round(mx * 1e9))
        low_ns = int(round((2.0 * mean - mx) * 1e9))
        for it in range(11):
            incl[0 + it * nn + k] = low_ns
            incl[11 * nn + it * nn + k] = max_ns
    return {"incl": incl, "block_offset": np.array([0, 11 * nn], np.uint64),
            "iter_counts": np.array([11, 11], np.uint32), "node_ids": np.arange(2, 8, dtype=np.uint32)}


def test_kat_savings_arithmetic():
    """acceptance.cpp:106-121: per-iteration savings, totals, grand total 28.083, speedup 0.3228."""
    cb = savings_fixture_cube()
    expect_savings = [1.687, 0.116, 0.211, 0.475, 0.061, 0.003]
    expect_total = [18.557, 1.276, 2.321, 5.225, 0.671, 0.033]
    grand = 0.0
    for k in range(6):
        row, _ = oracle.node_stats(cb, k)
        assert abs(row[2] - expect_savings[k]) <= 1e-9
        assert abs(row[3] - expect_total[k]) <= 1e-9
        grand += row[3]
    assert abs(grand - 28.083) <= 1e-9
    assert abs(grand / 87.0 - 0.3228) <= 5e-4


def test_kat_balance_ratio_and_cv():
    """test_diagnostics.cpp:57-91 through the oracle's outlier chain (one site)."""
    def ratio(v):
        vals = np.array([v], np.int64)
        return oracle.outliers(vals, np.zeros(len(v), np.uint32), 1, 0, -1e300)["site_ratio"][0]
    assert ratio([2, 2, 2]) == 1.0
    assert abs(ratio([1, 3]) - 2.0 / 3.0) <= 1e-15
    assert ratio([0, 0]) == 1.0
    assert abs(ratio([int(round((2 * 0.483 - 0.958) * 1e9)), int(0.958e9)]) - 0.504) <= 2e-3


# ---- golden vectors from the reference ----------------------------------------

@pytest.mark.parametrize("name", FIXTURES)
def test_window_oracle_matches_reference(name):
    g = load(name)
    tr = traces(g)
    n, n_ctx = len(g["pid"]), len(g["parent"])
    for i, (t0, t1) in enumerate(g["windows"]):
        o = oracle.window(tr, g["parent"], int(t0), int(t1))
        r = densify_window(g, i, n, n_ctx)
        for k in ("count", "sum", "min", "max", "mean", "excl", "incl"):
            assert np.array_equal(o[k], r[k]), f"{name} window {i}: {k}"
        for k in ("has", "ts", "ctx"):
            assert np.array_equal(o["carry"][k], r["carry"][k]), f"{name} window {i}: carry {k}"
        # ingest_traces rows == the linear-scan restatement (store.cpp:633-676)
        keep = (tr["ts"] >= t0) & (tr["ts"] < t1)
        pid_of = np.repeat(tr["pid"], np.diff(tr["off"]).astype(np.int64))
        assert np.array_equal(g[f"w{i}_rows_ts"], tr["ts"][keep])
        assert np.array_equal(g[f"w{i}_rows_ctx"], tr["ctx"][keep])
        assert np.array_equal(g[f"w{i}_rows_pid"], pid_of[keep])


@pytest.mark.parametrize("name", FIXTURES)
def test_cube_oracle_matches_reference(name):
    g = load(name)
    tr = traces(g)
    for i, a in enumerate(g["anchors"]):
        o = oracle.cube(tr, g["parent"], int(a))
        kept = o["iter_counts"] > 0
        assert np.array_equal(o["node_ids"], g[f"c{i}_node_ids"])
        assert np.array_equal(tr["pid"][kept], g[f"c{i}_trace_ids"])
        assert np.array_equal(tr["pid"][~kept], g[f"c{i}_skipped"])
        assert np.array_equal(o["iter_counts"][kept], g[f"c{i}_iter_counts"])
        for k in ("block_offset", "incl", "excl", "gap_incl", "gap_excl"):
            assert np.array_equal(o[k], g[f"c{i}_{k}"]), f"{name} anchor {a}: {k}"
        if not kept.any() or not int(g[f"c{i}_savings_ok"][0]):
            continue
        leaves = g[f"c{i}_leaves"]
        sav = g[f"c{i}_savings"].reshape(-1, 4)
        cv = g[f"c{i}_cv"].reshape(-1, 2)
        for j, leaf in enumerate(leaves):
            row, ok = oracle.node_stats(o, int(np.searchsorted(o["node_ids"], leaf)))
            assert_rel(row[:4], sav[j], 1e-9, f"{name} savings leaf {leaf}")
            assert ok == bool(g[f"c{i}_cv_ok"][j])
            if ok:
                assert_rel(row[4:], cv[j], 1e-9, f"{name} cv leaf {leaf}")


def test_congestion_oracle_matches_reference():
    """The z-score/top-k restatement on node means reproduces the reference's
    DBSCAN outlier group (workflows.cpp:478-539) and its balance ratios."""
    g = load("congestion_rpn2")
    hosts = [str(h) for h in g["hosts"]]
    n_nodes = len(hosts)
    o = oracle.outliers(g["site_values"], g["node_of_trace"], n_nodes, 0, 1.0)
    assert_rel(o["site_ratio"], g["ref_ratio"], 1e-9, "balance ratios")
    assert g["site_ctx"][o["worst"]] == g["ref_worst_ctx"][0]
    got = sorted(hosts[i] for i in o["selected"])
    assert got == [str(h) for h in g["ref_outliers"]] == [str(h) for h in g["truth_outliers"]]
    assert len(got) == 202
    # topology (topology.cpp:54-92): racks of the outlier hosts, ascending
    racks = {}
    for h in got:
        m = re.fullmatch(r"x(\d+)c(\d+)s(\d+)b(\d+)n(\d+)", h)
        racks[int(m.group(1))] = racks.get(int(m.group(1)), 0) + 1
    assert sorted(racks) == g["ref_racks"].tolist()
    assert [racks[r] for r in sorted(racks)] == g["ref_rack_nodes"].tolist()
    # top-k with k = |group| selects the same set
    o2 = oracle.outliers(g["site_values"], g["node_of_trace"], n_nodes, 202, -1e300)
    assert sorted(hosts[i] for i in o2["selected"]) == got


# ---- the C-ABI library (no compute calls without a GPU) -------------------------

def declared_symbols() -> list[str]:
    names = []
    for h in ("psg.h", "perfslice_gpu.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names += re.findall(r"\b(psg_[a-z_0-9]+)\s*\(", src)
    return sorted(set(names))


def test_c_abi_library_exports_every_declared_symbol():
    import ctypes

    from paper_2605_03561_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, f"libpsg.so lacks {missing}"
    assert set(syms) == set(_lib.EXPORTED), "ctypes binding out of sync with include/*.h"
    # pure host entry points are callable without a device
    lib.psg_version.restype = ctypes.c_char_p
    assert lib.psg_version().decode().endswith("sm100a")
    lib.psg_status_name.restype = ctypes.c_char_p
    assert lib.psg_status_name(13) == b"invalid_argument"


def test_context_open_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2605_03561_b200 import Context, PsgError
    with pytest.raises(PsgError) as e:
        Context(0)
    assert e.value.name == "internal"


def test_libpsg_is_sm100a_only():
    """The shipped cubin targets sm_100a (no PTX JIT fallback, no other arch)."""
    import subprocess

    from paper_2605_03561_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_suggest_anchor_oracle_matches_reference():
    """itermodel.cpp:45-109 on the first trace: the oracle's restatement picks
    the reference's anchor (or none, where the reference raises no_periodicity)."""
    for name in FIXTURES:
        g = load(name)
        assert oracle.suggest_anchor(traces(g), g["parent"], 0) == int(g["auto_anchor"][0]), name
    z = load("anchor_cases")
    for i in range(int(z["n_cases"][0])):
        tr = {k: z[f"case{i}_{k}"] for k in ("ts", "ctx", "off", "t_end", "pid")}
        assert oracle.suggest_anchor(tr, z["parent"], 0) == int(z[f"case{i}_anchor"][0]), i


def _fixture_pdb(g: dict) -> dict:
    rec = np.dtype([("ctx", "<u4"), ("metric", "<u2"), ("value", "<f8")])
    r = np.frombuffer(g["body"].tobytes(), dtype=rec)
    return {"pid": g["pid"], "rec_off": g["rec_off"], "ctx": r["ctx"].astype(np.uint32),
            "metric": r["metric"].astype(np.uint16), "value": r["value"].astype(np.float64)}


def test_profile_slice_oracle_matches_ingest_profiles():
    """read_slices / ingest_profiles restated (oracle.slices) == the reference's
    own rows, all contexts and a keep set + metric filter (tests/golden)."""
    g = load("profiles_rpn1")
    pdb = _fixture_pdb(g)
    for pre, cx, mt in (("all_", None, None), ("filt_", g["req_ctx"], [1])):
        o = oracle.slices(pdb, g["req_pids"], cx, mt)
        for k in ("pid", "ctx", "metric", "value"):
            assert np.array_equal(o[k], g[pre + k]), f"{pre}{k}"


def test_profile_congestion_oracle_matches_reference():
    """rank_vector + balance_ratio + node_correlate over profile records ==
    congestion_report's call-site ratios and worst site (tests/golden)."""
    g = load("profiles_rpn1")
    pdb = _fixture_pdb(g)
    meta = {"profiles": list(zip(g["prof_pid"].tolist(), g["prof_rank"].tolist(),
                                 g["prof_host"].tolist()))}
    o = oracle.profile_sites(pdb, meta, 1, g["site_ctx"])
    assert_rel(o["ratio"], g["ref_ratio"], 1e-12, "balance ratios")
    assert int(g["site_ctx"][o["worst"]]) == int(g["ref_worst_ctx"][0])


def _frame_inputs(seed: int, n: int):
    rng = np.random.default_rng(seed)
    a = rng.integers(-6, 6, n).astype(np.int64)
    b = rng.random(n)
    b[::7] = np.nan
    b[::11] = -0.0
    b[::13] = 0.0
    c = rng.integers(0, 4, n).astype(np.uint64)
    return a, b, c


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", range(3))
def test_frame_oracle_matches_reference(seed):
    """Stable multi-key argsort over NaN / +-0 / duplicate keys and the
    4096-block fold of reduce_sum / cumulative_sum, restated in numpy, equal
    the reference's frame::sort / reduce_sum / cumulative_sum bit for bit."""
    a, b, c = _frame_inputs(seed, 9000)
    for asc in (None, [True, False, True], [False, True, False]):
        assert np.array_equal(oracle.frame_argsort([a, b, c], asc), oracle.ref_frame_sort([a, b, c], asc))
    x = np.random.default_rng(seed).random(50_000) * 1e3 - 500
    tot, cs = oracle.frame_block_scan(x)
    assert tot == oracle.ref_frame_vec("reduce_sum", x)
    assert np.array_equal(cs, oracle.ref_frame_vec("cumsum", x))

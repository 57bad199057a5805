#!/usr/bin/env python
"""Writes the golden vectors under tests/golden/*.npz from the UNMODIFIED
reference (oracle/_ref, built by oracle/build_ref.sh from /root/reference).

Run here (the container that has /root/reference):
    python tests/golden/make_golden.py
The fixtures are small (< 1 MB in total) and committed; the tests that use
them (tests/test_oracle.py on CPU, tests/test_gpu_parity.py on the GPU) never
need /root/reference at run time.

Every fixture holds the INPUT (the trace set as SoA + the calling-context
tree) and the reference's OUTPUT for it:
  * window  — ingest_traces + dur glue + frame::group_aggregate +
              itermodel::rematerialize over [t0, t1)   (ref_harness.cpp refh_window)
  * cube    — itermodel::build_tri_model + savings_report + iteration_cv_report
              (refh_trimodel)
  * congestion — workflows::congestion_report JSON plus the per-rank site
              values the reference clusters (profile records == trace integrals)
"""
from __future__ import annotations

import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2605_03561_b200 import scenarios  # noqa: E402
from tests.helpers import random_cct, random_traces  # noqa: E402

WINDOW_KEYS = ("wa_pid", "wa_ctx", "wa_sum", "wa_min", "wa_max", "wa_mean", "wa_count", "carry_pid",
               "carry_has", "carry_ts", "carry_ctx", "rm_pid", "rm_ctx", "rm_incl", "rm_excl")
CUBE_KEYS = ("anchor", "node_ids", "trace_ids", "iter_counts", "skipped", "block_offset", "incl",
             "excl", "gap_incl", "gap_excl", "leaves", "savings", "savings_summary", "savings_ok",
             "cv", "cv_ok")


def trace_arrays(db: str) -> dict:
    tr = oracle.read_trace_db(db)
    meta = oracle.read_meta(db)
    return {"ts": tr["ts"], "ctx": tr["ctx"], "off": tr["off"], "t_end": tr["t_end"],
            "pid": tr["pid"], "parent": meta["parent"]}


def add_windows(out: dict, db: str, windows) -> None:
    out["windows"] = np.array(windows, np.uint64).reshape(-1, 2)
    for i, (t0, t1) in enumerate(windows):
        r = oracle.ref_window(db, int(t0), int(t1), rows=True)
        for k in WINDOW_KEYS + ("rows_pid", "rows_ts", "rows_ctx"):
            out[f"w{i}_{k}"] = r[k]


def add_cubes(out: dict, db: str, anchors) -> None:
    out["anchors"] = np.array(anchors, np.int64)
    for i, a in enumerate(anchors):
        r = oracle.ref_trimodel(db, int(a))
        for k in CUBE_KEYS:
            out[f"c{i}_{k}"] = r[k]


def auto_anchor(db: str) -> np.ndarray:
    """suggest_anchor on the first trace (itermodel.cpp:253-255); 0xFFFFFFFF
    where the reference raises no_periodicity (or empty_input)."""
    try:
        return oracle.ref_trimodel(db, -1)["anchor"]
    except RuntimeError:
        return np.array([0xFFFFFFFF], np.uint32)


def iterative_fixture(name: str, cfg: dict, anchors=(1,)) -> None:
    with tempfile.TemporaryDirectory() as d:
        oracle.ref_generate(cfg, d)
        out = trace_arrays(d)
        T = int(out["t_end"].max())
        add_windows(out, d, [(T // 4, 3 * T // 4), (0, T + 1), (T // 3, T // 3)])
        add_cubes(out, d, anchors)
        out["auto_anchor"] = auto_anchor(d)
        out["config"] = np.frombuffer(json.dumps(cfg).encode(), np.uint8)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)


def random_fixture(name: str, seed: int) -> None:
    rng = np.random.default_rng(1000 + seed)
    n_ctx = int(rng.integers(3, 24))
    parent = random_cct(rng, n_ctx)
    tr = random_traces(rng, int(rng.integers(2, 24)), n_ctx, int(rng.integers(1, 300)),
                       ctx_pool=int(rng.integers(2, n_ctx + 1)), dup_prob=float(rng.random()) * 0.6)
    with tempfile.TemporaryDirectory() as d:
        oracle.ref_write_traces(tr, parent, d)
        out = {k: tr[k] for k in ("ts", "ctx", "off", "t_end", "pid")}
        out["parent"] = parent
        T = int(tr["t_end"].max()) if len(tr["t_end"]) else 10
        add_windows(out, d, [(0, T + 1), (T // 3, 2 * T // 3), (T // 2, T // 2), (T // 5, T // 5 + 7)])
        add_cubes(out, d, sorted({0, 1, int(rng.integers(0, n_ctx)), n_ctx - 1}))
        out["auto_anchor"] = auto_anchor(d)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)


def kat_single_segment() -> None:
    """test_itermodel.cpp:77-85: root -> mid -> leaf (+ sibling); one event
    {100, leaf} over [100, 105) gives leaf (5,5), mid (5,0), root (5,0)."""
    parent = np.array([0xFFFFFFFF, 0, 1, 0], np.uint32)
    tr = {"ts": np.array([100], np.uint64), "ctx": np.array([2], np.uint32),
          "off": np.array([0, 1], np.uint64), "t_end": np.array([105], np.uint64),
          "pid": np.array([1], np.uint32)}
    with tempfile.TemporaryDirectory() as d:
        oracle.ref_write_traces(tr, parent, d)
        out = dict(tr)
        out["parent"] = parent
        add_windows(out, d, [(100, 105)])
        np.savez_compressed(os.path.join(HERE, "kat_single_segment.npz"), **out)


def anchor_cases() -> None:
    """suggest_anchor on hand-shaped traces: nested periodic loops (the most
    covered periodic context wins), exact ties in covered time (smallest id),
    jittered gaps around the 0.2 CV cut, repeated timestamps."""
    rng = np.random.default_rng(77)
    out = {}
    cases = []
    # ctx: 0 root, 1 outer, 2 inner, 3 leafA (under inner), 4 leafB (under outer), 5 other (root)
    parent = np.array([0xFFFFFFFF, 0, 1, 2, 1, 0, 2, 4], np.uint32)
    for case in range(8):
        ts, cx = [], []
        t = int(rng.integers(0, 50))
        jit = [0.0, 0.05, 0.15, 0.3, 0.5, 0.0, 0.1, 0.25][case]
        for it in range(int(rng.integers(4, 12))):
            ts.append(t); cx.append(1)
            for j in range(int(rng.integers(1, 4))):
                ts.append(t); cx.append(2)
                d = max(1, int(100 * (1 + jit * rng.standard_normal())))
                ts.append(t); cx.append(3 if case % 2 else 6)
                t += d
                ts.append(t); cx.append(7 if case == 5 else 4)
                t += max(1, int(40 * (1 + jit * rng.standard_normal())))
            ts.append(t); cx.append(0)
            t += int(rng.integers(0, 3)) * (0 if case == 5 else 1)
            if case in (6, 7):
                ts.append(t); cx.append(5)
                t += 30
        t_end = t + int(rng.integers(0, 20))
        tr = {"ts": np.array(ts, np.uint64), "ctx": np.array(cx, np.uint32),
              "off": np.array([0, len(ts)], np.uint64), "t_end": np.array([t_end], np.uint64),
              "pid": np.array([1], np.uint32)}
        with tempfile.TemporaryDirectory() as d:
            oracle.ref_write_traces(tr, parent, d)
            a = auto_anchor(d)
        for k, v in tr.items():
            out[f"case{case}_{k}"] = v
        out[f"case{case}_anchor"] = a
        cases.append(int(a[0]))
    out["parent"] = parent
    out["n_cases"] = np.array([len(cases)])
    np.savez_compressed(os.path.join(HERE, "anchor_cases.npz"), **out)


def congestion_fixture(name: str, ranks_per_node: int, seed: int) -> None:
    cfg = scenarios.aurora(ranks_per_node=ranks_per_node, seed=seed)
    with tempfile.TemporaryDirectory() as d:
        truth = oracle.ref_generate(cfg, d)
        tr = oracle.read_trace_db(d)
        meta = oracle.read_meta(d)
        rep = json.loads(oracle.ref_congestion_report(d))
        sites = np.array(truth["callsite_ctx"], np.uint32)
        # per-rank inclusive ns of each call site over the whole trace (the
        # profile record cputime(i) the reference reads, synthgen.cpp:79-103)
        w = oracle.window(tr, meta["parent"], 0, 2**64 - 1, clamp_tend=True)
        hosts = sorted({h for (_, r, h) in meta["profiles"] if r >= 0})
        hidx = {h: i for i, h in enumerate(hosts)}
        rank_host = {}
        for (_, r, h) in meta["profiles"]:
            if r >= 0 and r not in rank_host:
                rank_host[r] = h
        prof = {p: r for (p, r, _) in meta["profiles"]}
        node_of_trace = np.array([hidx[rank_host[prof[int(p)]]] for p in tr["pid"]], np.uint32)
        out = {
            "site_ctx": sites, "site_values": np.ascontiguousarray(w["incl"][:, sites].T),
            "node_of_trace": node_of_trace, "hosts": np.array(hosts),
            "ref_ratio": np.array([s["balance_ratio"] for s in rep["callsites"]], np.float64),
            "ref_worst_ctx": np.array([rep["worst"]["ctx_id"]], np.uint32),
            "ref_outliers": np.array(sorted(rep["outlier_group"]["hostnames"])),
            "ref_racks": np.array([r["rack"] for r in rep["topology"]["racks"]], np.uint32),
            "ref_rack_nodes": np.array([r["nodes"] for r in rep["topology"]["racks"]], np.uint32),
            "truth_outliers": np.array(sorted(truth["outlier_hostnames"])),
            "report": np.frombuffer(json.dumps(rep).encode(), np.uint8),
        }
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)


def profile_fixture(name: str, ranks_per_node: int, seed: int) -> None:
    """profile.db of the aurora-like scenario with the reference's
    ingest_profiles slices (all / filtered) and congestion_report ratios."""
    cfg = scenarios.aurora(ranks_per_node=ranks_per_node, seed=seed)
    with tempfile.TemporaryDirectory() as d:
        truth = oracle.ref_generate(cfg, d)
        meta = oracle.read_meta(d)
        pdb = oracle.read_profile_db(d)
        rep = json.loads(oracle.ref_congestion_report(d))
        pids = [p for (p, _, _) in meta["profiles"]]
        some = pids[::7]
        ctxs = [0, 1] + list(truth["callsite_ctx"])
        all_rows = oracle.ref_slices(d, some)
        filt = oracle.ref_slices(d, some, sorted(ctxs), [1])
        out = {
            "body": pdb["body"], "rec_off": pdb["rec_off"], "pid": pdb["pid"],
            "prof_pid": np.array(pids, np.uint32),
            "prof_rank": np.array([r for (_, r, _) in meta["profiles"]], np.int32),
            "prof_host": np.array([h for (_, _, h) in meta["profiles"]]),
            "req_pids": np.array(some, np.uint32), "req_ctx": np.array(sorted(ctxs), np.uint32),
            "site_ctx": np.array(truth["callsite_ctx"], np.uint32),
            "ref_ratio": np.array([s["balance_ratio"] for s in rep["callsites"]], np.float64),
            "ref_worst_ctx": np.array([rep["worst"]["ctx_id"]], np.uint32),
            "ref_outliers": np.array(sorted(rep["outlier_group"]["hostnames"])),
        }
        for k, v in all_rows.items():
            out["all_" + k] = v
        for k, v in filt.items():
            out["filt_" + k] = v
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)


def main() -> None:
    if not oracle.ref_available():
        raise SystemExit("oracle/_ref missing: run oracle/build_ref.sh first")
    kat_single_segment()
    iterative_fixture("small_iter", scenarios.small(seed=52, n_ranks=4, n_iterations=7, jitter=0.1),
                      anchors=(1, 0))
    iterative_fixture("gamess_like", scenarios.iterative(12, 9, n_kernels=6, seed=9, spread="gamess"),
                      anchors=(1,))
    for s in range(4):
        random_fixture(f"random_{s}", s)
    anchor_cases()
    congestion_fixture("congestion_rpn2", ranks_per_node=2, seed=2025)
    profile_fixture("profiles_rpn1", ranks_per_node=1, seed=2025)
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f"{f:28s} {os.path.getsize(os.path.join(HERE, f)):8d} B")


if __name__ == "__main__":
    main()

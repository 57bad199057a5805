"""TEST INFRASTRUCTURE ONLY (checker, never the thing measured or shipped).

Python bindings of
  * oracle/liboracle.so       — the CPU restatement (oracle/psg_oracle.c);
  * oracle/_ref/libps_refharness.so — the UNMODIFIED reference core plus our
    harness (oracle/ref_harness.cpp), built by oracle/build_ref.sh.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import struct
import subprocess
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_DIR = os.path.join(HERE, "_ref")
REF_SO = os.path.join(REF_DIR, "libps_refharness.so")

U8P, U32P, U64P = C.POINTER(C.c_uint8), C.POINTER(C.c_uint32), C.POINTER(C.c_uint64)
I32P, I64P, F64P = C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_double)


def _p(a, t):
    return None if a is None else a.ctypes.data_as(C.POINTER(t))


def build_oracle() -> str:
    if not os.path.exists(ORACLE_SO) or os.path.getmtime(ORACLE_SO) < os.path.getmtime(
            os.path.join(HERE, "psg_oracle.c")):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return ORACLE_SO


_orc = None


def orc():
    global _orc
    if _orc is None:
        lib = C.CDLL(build_oracle())
        lib.orc_window.restype = None
        lib.orc_window.argtypes = [U64P, U64P, U32P, C.c_uint32, U32P, C.c_uint32, C.c_uint64,
                                   C.c_uint64, U64P, U64P, I64P, I64P, I64P, F64P, I64P, I64P, U8P, U64P,
                                   U32P]
        lib.orc_iter_counts.restype = None
        lib.orc_iter_counts.argtypes = [U64P, U64P, U32P, U64P, C.c_uint32, U32P, C.c_uint32,
                                        C.c_uint32, U32P]
        lib.orc_subtree.restype = C.c_uint32
        lib.orc_subtree.argtypes = [U32P, C.c_uint32, C.c_uint32, U32P]
        lib.orc_cube.restype = None
        lib.orc_cube.argtypes = [U64P, U64P, U32P, U64P, C.c_uint32, U32P, C.c_uint32, C.c_uint32,
                                 I64P, I64P, I64P, I64P]
        lib.orc_node_stats.restype = None
        lib.orc_node_stats.argtypes = [I64P, U64P, U32P, C.c_uint32, C.c_uint32, C.c_uint32, F64P,
                                       C.POINTER(C.c_int)]
        lib.orc_outliers.restype = C.c_uint32
        lib.orc_outliers.argtypes = [I64P, C.c_uint32, C.c_uint32, U32P, C.c_uint32, C.c_uint32,
                                     C.c_double, F64P, U32P, F64P, F64P, U32P]
        lib.orc_suggest_anchor.restype = C.c_uint32
        lib.orc_suggest_anchor.argtypes = [U64P, U32P, C.c_uint64, C.c_uint64, U32P, C.c_uint32,
                                           C.c_uint32, C.c_double]
        _orc = lib
    return _orc


# ---- oracle restatement wrappers -------------------------------------------

def window(tr: dict, parent, t0: int, t1: int, clamp_tend: bool = False) -> dict:
    n = len(tr["off"]) - 1
    parent = np.ascontiguousarray(parent, np.uint32)
    nc = len(parent)
    out = {k: np.zeros((n, nc), dt) for k, dt in [
        ("count", np.uint64), ("sum", np.int64), ("min", np.int64), ("max", np.int64),
        ("mean", np.float64), ("excl", np.int64), ("incl", np.int64)]}
    has, cts, cctx = np.zeros(n, np.uint8), np.zeros(n, np.uint64), np.zeros(n, np.uint32)
    orc().orc_window(_p(tr["off"], C.c_uint64), _p(tr["ts"], C.c_uint64), _p(tr["ctx"], C.c_uint32),
                     n, _p(parent, C.c_uint32), nc, t0, t1,
                     _p(np.ascontiguousarray(tr["t_end"], np.uint64), C.c_uint64) if clamp_tend else None,
                     _p(out["count"], C.c_uint64),
                     _p(out["sum"], C.c_int64), _p(out["min"], C.c_int64), _p(out["max"], C.c_int64),
                     _p(out["mean"], C.c_double), _p(out["excl"], C.c_int64),
                     _p(out["incl"], C.c_int64), _p(has, C.c_uint8), _p(cts, C.c_uint64),
                     _p(cctx, C.c_uint32))
    out["carry"] = {"has": has, "ts": cts, "ctx": cctx}
    return out


def cube(tr: dict, parent, anchor: int) -> dict:
    n = len(tr["off"]) - 1
    parent = np.ascontiguousarray(parent, np.uint32)
    nc = len(parent)
    ic = np.zeros(n, np.uint32)
    args = (_p(tr["off"], C.c_uint64), _p(tr["ts"], C.c_uint64), _p(tr["ctx"], C.c_uint32),
            _p(tr["t_end"], C.c_uint64), n, _p(parent, C.c_uint32), nc, anchor)
    orc().orc_iter_counts(*args, _p(ic, C.c_uint32))
    nn = orc().orc_subtree(_p(parent, C.c_uint32), nc, anchor, None)
    node_ids = np.zeros(nn, np.uint32)
    orc().orc_subtree(_p(parent, C.c_uint32), nc, anchor, _p(node_ids, C.c_uint32))
    kept = ic[ic > 0]
    cells = int(kept.astype(np.uint64).sum()) * nn
    incl, excl = np.zeros(cells, np.int64), np.zeros(cells, np.int64)
    gi, ge = np.zeros(len(kept) * nn, np.int64), np.zeros(len(kept) * nn, np.int64)
    orc().orc_cube(*args, _p(incl, C.c_int64), _p(excl, C.c_int64), _p(gi, C.c_int64),
                   _p(ge, C.c_int64))
    bo = np.zeros(len(kept), np.uint64)
    if len(kept):
        bo[1:] = np.cumsum(kept.astype(np.uint64) * nn)[:-1]
    return {"node_ids": node_ids, "iter_counts": ic, "block_offset": bo, "incl": incl,
            "excl": excl, "gap_incl": gi, "gap_excl": ge}


def suggest_anchor(tr: dict, parent, t: int = 0, min_iters: int = 3, cv_max: float = 0.2) -> int:
    """suggest_anchor on trace t (0xFFFFFFFF: no periodic context)."""
    parent = np.ascontiguousarray(parent, np.uint32)
    b, e = int(tr["off"][t]), int(tr["off"][t + 1])
    ts = np.ascontiguousarray(tr["ts"][b:e], np.uint64)
    cx = np.ascontiguousarray(tr["ctx"][b:e], np.uint32)
    return int(orc().orc_suggest_anchor(_p(ts, C.c_uint64), _p(cx, C.c_uint32), e - b,
                                        int(tr["t_end"][t]), _p(parent, C.c_uint32), len(parent),
                                        min_iters, cv_max))


def node_stats(cb: dict, npos: int) -> tuple[np.ndarray, bool]:
    kept = cb["iter_counts"][cb["iter_counts"] > 0].astype(np.uint32)
    nn = len(cb["node_ids"])
    out = np.zeros(6, np.float64)
    ok = C.c_int(0)
    bo = np.ascontiguousarray(cb["block_offset"], np.uint64)
    orc().orc_node_stats(_p(cb["incl"], C.c_int64), _p(bo, C.c_uint64), _p(kept, C.c_uint32),
                         len(kept), nn, npos, _p(out, C.c_double), C.byref(ok))
    return out, bool(ok.value)


def outliers(values: np.ndarray, node_of_rank, n_nodes: int, top_k: int, z_min: float) -> dict:
    values = np.ascontiguousarray(values, np.int64)
    ns, nr = values.shape
    nor = np.ascontiguousarray(node_of_rank, np.uint32)
    ratio = np.zeros(ns)
    worst = C.c_uint32(0)
    mean, z = np.zeros(n_nodes), np.zeros(n_nodes)
    sel = np.zeros(n_nodes, np.uint32)
    k = orc().orc_outliers(_p(values, C.c_int64), ns, nr, _p(nor, C.c_uint32), n_nodes, top_k,
                           z_min, _p(ratio, C.c_double), C.byref(worst), _p(mean, C.c_double),
                           _p(z, C.c_double), _p(sel, C.c_uint32))
    return {"site_ratio": ratio, "worst": worst.value, "node_mean": mean, "node_z": z,
            "selected": sel[:k]}


# ---- the reference (oracle/_ref) --------------------------------------------

_ref = None


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not ref_available():
            raise RuntimeError(f"{REF_SO} missing: run oracle/build_ref.sh where /root/reference exists")
        lib = C.CDLL(REF_SO)
        lib.refh_last_error.restype = C.c_char_p
        lib.refh_free.argtypes = [C.c_void_p]
        lib.refh_default_jobs.restype = C.c_uint
        lib.refh_generate.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p)]
        lib.refh_write_traces.argtypes = [C.c_char_p, U32P, C.c_uint32, U32P, U64P, U64P, U32P,
                                          U64P, C.c_uint32]
        lib.refh_window.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64, C.c_uint, C.c_char_p, C.c_int]
        lib.refh_trimodel.argtypes = [C.c_char_p, C.c_int64, C.c_uint, C.c_double, C.c_char_p]
        lib.refh_iterations_report.argtypes = [C.c_char_p, C.c_char_p, C.c_double, C.c_int, C.c_uint,
                                               C.POINTER(C.c_void_p)]
        lib.refh_congestion_report.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_uint,
                                               C.c_double, C.c_double, C.c_int, C.c_uint,
                                               C.POINTER(C.c_void_p)]
        for f in ("refh_time_window", "refh_time_trimodel", "refh_time_query", "refh_time_congestion"):
            getattr(lib, f).restype = C.c_double
        lib.refh_time_window.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64, C.c_uint, C.c_uint]
        lib.refh_time_trimodel.argtypes = [C.c_char_p, C.c_int64, C.c_uint, C.c_uint]
        lib.refh_time_query.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64, C.c_int64, C.c_uint,
                                        C.c_uint]
        lib.refh_time_congestion.argtypes = [C.c_char_p, C.c_uint, C.c_uint]
        _ref = lib
    return _ref


def _chk(rc):
    if rc != 0:
        raise RuntimeError(f"reference harness error {rc}: {ref().refh_last_error().decode()}")


def _take(ptr: C.c_void_p) -> str:
    s = C.cast(ptr, C.c_char_p).value.decode()
    ref().refh_free(ptr)
    return s


def ref_generate(cfg: dict, out_dir: str) -> dict:
    """workflows::generate_database: writes meta.bin/profile.db/trace.db/truth.json."""
    p = C.c_void_p()
    _chk(ref().refh_generate(json.dumps(cfg).encode(), out_dir.encode(), C.byref(p)))
    return json.loads(_take(p))


def ref_write_traces(tr: dict, parent, out_dir: str) -> None:
    """store::write_database of raw SoA traces (one profile per trace)."""
    parent = np.ascontiguousarray(parent, np.uint32)
    a = {k: np.ascontiguousarray(tr[k], dt) for k, dt in
         (("pid", np.uint32), ("off", np.uint64), ("ts", np.uint64), ("ctx", np.uint32),
          ("t_end", np.uint64))}
    _chk(ref().refh_write_traces(out_dir.encode(), _p(parent, C.c_uint32), len(parent),
                                 _p(a["pid"], C.c_uint32), _p(a["off"], C.c_uint64),
                                 _p(a["ts"], C.c_uint64), _p(a["ctx"], C.c_uint32),
                                 _p(a["t_end"], C.c_uint64), len(a["pid"])))


def _load_bins(d: str, spec: dict) -> dict:
    return {k: np.fromfile(os.path.join(d, k + ".bin"), dtype=dt) for k, dt in spec.items()}


def ref_window(db: str, t0: int, t1: int, jobs: int = 1, rows: bool = False) -> dict:
    with tempfile.TemporaryDirectory() as d:
        _chk(ref().refh_window(db.encode(), t0, t1, jobs, d.encode(), int(rows)))
        spec = {"wa_pid": np.uint64, "wa_ctx": np.uint64, "wa_sum": np.int64, "wa_min": np.int64,
                "wa_max": np.int64, "wa_mean": np.float64, "wa_count": np.uint64,
                "carry_pid": np.uint32, "carry_has": np.uint8, "carry_ts": np.uint64,
                "carry_ctx": np.uint32, "rm_pid": np.uint32, "rm_ctx": np.uint32,
                "rm_incl": np.int64, "rm_excl": np.int64}
        if rows:
            spec.update({"rows_pid": np.uint32, "rows_ts": np.uint64, "rows_ctx": np.uint32})
        return _load_bins(d, spec)


def ref_trimodel(db: str, anchor: int, jobs: int = 1, total_time: float = 0.0) -> dict:
    with tempfile.TemporaryDirectory() as d:
        _chk(ref().refh_trimodel(db.encode(), anchor, jobs, total_time, d.encode()))
        return _load_bins(d, {
            "anchor": np.uint32, "node_ids": np.uint32, "trace_ids": np.uint32,
            "iter_counts": np.uint32, "skipped": np.uint32, "block_offset": np.uint64,
            "incl": np.int64, "excl": np.int64, "gap_incl": np.int64, "gap_excl": np.int64,
            "leaves": np.uint32, "savings": np.float64, "savings_summary": np.float64,
            "savings_ok": np.int32, "cv": np.float64, "cv_ok": np.int32})


def ref_iterations_report(db: str, anchor: str = "auto", total_time: float = 0.0,
                          json_fmt: bool = True, jobs: int = 1) -> str:
    p = C.c_void_p()
    _chk(ref().refh_iterations_report(db.encode(), anchor.encode(), total_time, int(json_fmt), jobs,
                                      C.byref(p)))
    return _take(p)


def ref_congestion_report(db: str, glob: str = "MPI_*", method: str = "dbscan", k: int = 2,
                          eps: float = 0.0, min_share: float = 0.01, json_fmt: bool = True,
                          jobs: int = 1) -> str:
    p = C.c_void_p()
    _chk(ref().refh_congestion_report(db.encode(), glob.encode(), method.encode(), k, eps, min_share,
                                      int(json_fmt), jobs, C.byref(p)))
    return _take(p)


def ref_localize(outliers, universe) -> dict:
    """topology::localize_outliers (topology.cpp:54-92) as its JSON report;
    raises RuntimeError with the reference's parse_error message on a bad name."""
    o = [h.encode() for h in outliers]
    u = [h.encode() for h in universe]
    oa = (C.c_char_p * max(1, len(o)))(*o)
    ua = (C.c_char_p * max(1, len(u)))(*u)
    p = C.c_void_p()
    lib = ref()
    lib.refh_localize.argtypes = [C.POINTER(C.c_char_p), C.c_size_t, C.POINTER(C.c_char_p), C.c_size_t,
                                  C.POINTER(C.c_void_p)]
    _chk(lib.refh_localize(oa, len(o), ua, len(u), C.byref(p)))
    return json.loads(_take(p))


def ref_slices(db: str, pids, ctx_ids=None, metric_ids=None, jobs: int = 1) -> dict:
    """The reference's ingest_profiles (ingest.cpp:155-176) through oracle/_ref."""
    p = np.ascontiguousarray(pids, np.uint32)
    cx = np.ascontiguousarray([] if ctx_ids is None else ctx_ids, np.uint32)
    mt = np.ascontiguousarray([] if metric_ids is None else metric_ids, np.uint16)
    lib = ref()
    lib.refh_slices.argtypes = [C.c_char_p, C.POINTER(C.c_uint32), C.c_uint32, C.POINTER(C.c_uint32),
                                C.c_uint32, C.c_int, C.POINTER(C.c_uint16), C.c_uint32, C.c_uint,
                                C.c_char_p]
    with tempfile.TemporaryDirectory() as d:
        _chk(lib.refh_slices(db.encode(), _p(p, C.c_uint32), len(p), _p(cx, C.c_uint32), len(cx),
                             int(ctx_ids is None), _p(mt, C.c_uint16), len(mt), jobs, d.encode()))
        return _load_bins(d, {"pid": np.uint32, "ctx": np.uint32, "metric": np.uint16,
                              "value": np.float64})


def read_profile_db(db: str) -> dict:
    """Tiny independent reader of profile.db (store.hpp:11-14): per profile its
    id and the packed 14-byte records, plus the whole body as bytes."""
    raw = open(os.path.join(db, "profile.db"), "rb").read()
    assert raw[:4] == b"HPPR"
    n = struct.unpack_from("<I", raw, 8)[0]
    pids, offs, cnts = [], [], []
    for i in range(n):
        pid, off, cnt = struct.unpack_from("<IQQ", raw, 12 + 20 * i)
        pids.append(pid), offs.append(off), cnts.append(cnt)
    rec = np.dtype([("ctx", "<u4"), ("metric", "<u2"), ("value", "<f8")])
    body = b"".join(raw[o:o + 14 * c] for o, c in zip(offs, cnts))
    recs = np.frombuffer(body, dtype=rec)
    return {"pid": np.array(pids, np.uint32),
            "rec_off": np.concatenate([[0], np.cumsum(cnts)]).astype(np.uint64),
            "body": np.frombuffer(body, np.uint8), "ctx": recs["ctx"].astype(np.uint32),
            "metric": recs["metric"].astype(np.uint16), "value": recs["value"].astype(np.float64)}


def slices(pdb: dict, pids, ctx_ids=None, metric_ids=None) -> dict:
    """CPU restatement of read_slices (ingest.cpp:122-153) over read_profile_db
    arrays: sorted unique profiles, records in order, filtered by ctx and metric
    (records are ctx-sorted, so the reference's per-ctx binary-search runs
    visit them in record order, store.cpp:598-628)."""
    out = {"pid": [], "ctx": [], "metric": [], "value": []}
    cset = None if ctx_ids is None else set(int(c) for c in ctx_ids)
    mset = None if metric_ids is None else set(int(m) for m in metric_ids)
    for p in sorted(set(int(x) for x in pids)):
        i = int(np.searchsorted(pdb["pid"], p))
        assert i < len(pdb["pid"]) and pdb["pid"][i] == p, f"profile {p} not in database"
        a, b = int(pdb["rec_off"][i]), int(pdb["rec_off"][i + 1])
        for r in range(a, b):
            c, m = int(pdb["ctx"][r]), int(pdb["metric"][r])
            if (cset is None or c in cset) and (mset is None or m in mset):
                out["pid"].append(p), out["ctx"].append(c), out["metric"].append(m)
                out["value"].append(float(pdb["value"][r]))
    return {"pid": np.array(out["pid"], np.uint32), "ctx": np.array(out["ctx"], np.uint32),
            "metric": np.array(out["metric"], np.uint16), "value": np.array(out["value"], np.float64)}


def profile_sites(pdb: dict, meta: dict, metric: int, sites) -> dict:
    """congestion_report's numeric core over profile records
    (workflows.cpp:42-62, 442-471; diagnostics.cpp:10-19, 378-403): per site the
    rank_vector (rank profiles sorted by (rank, value), absent records as 0),
    its balance ratio, the worst (first minimal) site and the node means of
    its values over the sorted host list."""
    ranks = {int(pid): (int(r), h) for (pid, r, h) in meta["profiles"]}
    rank_host = {}
    for (pid, r, h) in meta["profiles"]:
        if r >= 0 and r not in rank_host:
            rank_host[r] = h
    ratios, vectors = [], []
    for s in sites:
        by_profile = {}
        sl = slices(pdb, [p for p in pdb["pid"] if ranks.get(int(p), (-1, ""))[0] >= 0], [s], [metric])
        for p, v in zip(sl["pid"], sl["value"]):
            by_profile[int(p)] = float(v)
        rv = sorted((ranks[int(p)][0], by_profile.get(int(p), 0.0)) for p in pdb["pid"]
                    if ranks.get(int(p), (-1, ""))[0] >= 0)
        vals = [v for _, v in rv]
        mx, sm = vals[0], 0.0
        for v in vals:
            mx, sm = max(mx, v), sm + v
        ratios.append(1.0 if mx == 0.0 else sm / len(vals) / mx)
        vectors.append(rv)
    w = min(range(len(sites)), key=lambda i: (ratios[i], i))
    acc = {}
    for r, v in vectors[w]:
        a = acc.setdefault(rank_host[r], [0.0, 0])
        a[0] += v
        a[1] += 1
    hosts = sorted(acc)
    return {"ratio": np.array(ratios), "worst": w, "hosts": hosts,
            "node_mean": np.array([acc[h][0] / acc[h][1] for h in hosts])}


def read_trace_db(db: str) -> dict:
    """Tiny independent reader of trace.db (format store.hpp:15-18) for tests."""
    raw = np.fromfile(os.path.join(db, "trace.db"), dtype=np.uint8)
    n = int(raw[8:12].view(np.uint32)[0])
    idx = raw[12:12 + 36 * n].reshape(n, 36)
    pid = idx[:, 0:4].copy().view(np.uint32).ravel()
    off = idx[:, 4:12].copy().view(np.uint64).ravel()
    cnt = idx[:, 12:20].copy().view(np.uint64).ravel()
    t_end = idx[:, 28:36].copy().view(np.uint64).ravel()
    body_start = 12 + 36 * n
    total = int(cnt.sum())
    body = raw[body_start:body_start + 12 * total].reshape(total, 12) if total else np.zeros((0, 12), np.uint8)
    assert n == 0 or int(off[0]) == body_start
    ts = body[:, 0:8].copy().view(np.uint64).ravel()
    cx = body[:, 8:12].copy().view(np.uint32).ravel()
    offs = np.zeros(n + 1, np.uint64)
    offs[1:] = np.cumsum(cnt)
    return {"ts": ts, "ctx": cx, "off": offs, "t_end": t_end, "pid": pid,
            "body": raw[body_start:body_start + 12 * total]}


def read_meta(db: str) -> dict:
    """meta.bin (store.hpp:8-12): contexts (parent, kind, name) and profiles."""
    b = open(os.path.join(db, "meta.bin"), "rb").read()
    pos = 8

    def u(fmt, n):
        nonlocal pos
        v = np.frombuffer(b, dtype=fmt, count=1, offset=pos)[0]
        pos += n
        return int(v)

    def s():
        nonlocal pos
        ln = u(np.uint16, 2)
        r = b[pos:pos + ln].decode()
        pos += ln
        return r

    metrics = []
    for _ in range(u(np.uint32, 4)):
        mid = u(np.uint32, 4); scope = u(np.uint8, 1); name = s(); s()
        metrics.append((mid, scope, name))
    profiles = []
    for _ in range(u(np.uint32, 4)):
        pid = u(np.uint32, 4); rank = u(np.int32, 4); u(np.int32, 4); host = s(); u(np.uint64, 8)
        profiles.append((pid, rank, host))
    parent, names = [], []
    for _ in range(u(np.uint32, 4)):
        u(np.uint32, 4); parent.append(u(np.uint32, 4)); u(np.uint8, 1); names.append(s())
    return {"parent": np.array(parent, np.uint32), "names": names, "profiles": profiles,
            "metrics": metrics}


# ---- frame operators (frame.cpp) --------------------------------------------
_FRAME_DT = {np.dtype(np.int64): 0, np.dtype(np.uint64): 1, np.dtype(np.float64): 2}
FRAME_OPS = {"lt": 0, "le": 1, "eq": 2, "ge": 3, "gt": 4, "ne": 5}
FRAME_AGGS = {"sum": 0, "min": 1, "max": 2, "mean": 3, "count": 4}


def _ptrs(cols):
    arr = (C.c_void_p * max(1, len(cols)))(*[c.ctypes.data for c in cols])
    dts = (C.c_int * max(1, len(cols)))(*[_FRAME_DT[c.dtype] for c in cols])
    return arr, dts


def ref_frame_sort(keys, ascending=None, jobs: int = 1) -> np.ndarray:
    """The reference's frame::sort permutation (oracle/_ref)."""
    keys = [np.ascontiguousarray(k) for k in keys]
    n = len(keys[0])
    arr, dts = _ptrs(keys)
    asc = None if ascending is None else np.array([1 if a else 0 for a in ascending], np.uint8)
    perm = np.empty(max(1, n), np.uint64)
    _chk(ref().refh_frame_sort(C.c_uint64(n), len(keys), dts, arr,
                               asc.ctypes.data_as(C.c_void_p) if asc is not None else None, jobs,
                               perm.ctypes.data_as(C.c_void_p)))
    return perm[:n]


def ref_frame_group(keys, src, fn: str, jobs: int = 1):
    keys = [np.ascontiguousarray(k) for k in keys]
    src = np.ascontiguousarray(src)
    n = len(src)
    arr, dts = _ptrs(keys)
    ng = C.c_uint64()
    lib = ref()
    _chk(lib.refh_frame_group(C.c_uint64(n), len(keys), dts, arr, _FRAME_DT[src.dtype], C.c_void_p(src.ctypes.data),
                              FRAME_AGGS[fn], jobs, C.byref(ng), None, None))
    g = ng.value
    kout = [np.empty(max(1, g), k.dtype) for k in keys]
    odt = np.float64 if fn == "mean" else (np.uint64 if fn == "count" else src.dtype)
    agg = np.empty(max(1, g), odt)
    karr = (C.c_void_p * max(1, len(keys)))(*[k.ctypes.data for k in kout])
    _chk(lib.refh_frame_group(C.c_uint64(n), len(keys), dts, arr, _FRAME_DT[src.dtype], C.c_void_p(src.ctypes.data),
                              FRAME_AGGS[fn], jobs, C.byref(ng), karr, C.c_void_p(agg.ctypes.data)))
    return [k[:g] for k in kout], agg[:g]


def ref_frame_filter(col, op: str, literal, jobs: int = 1) -> np.ndarray:
    col = np.ascontiguousarray(col)
    lit = np.array([literal], col.dtype)
    m = C.c_uint64()
    idx = np.empty(max(1, len(col)), np.uint64)
    _chk(ref().refh_frame_filter(C.c_uint64(len(col)), _FRAME_DT[col.dtype], C.c_void_p(col.ctypes.data),
                                 FRAME_OPS[op], C.c_void_p(lit.ctypes.data), jobs, C.byref(m),
                                 C.c_void_p(idx.ctypes.data)))
    return idx[:m.value]


def ref_frame_merge(lkeys, rkeys, jobs: int = 1):
    lkeys = [np.ascontiguousarray(k) for k in lkeys]
    rkeys = [np.ascontiguousarray(k) for k in rkeys]
    la, dts = _ptrs(lkeys)
    ra, _ = _ptrs(rkeys)
    m = C.c_uint64()
    lib = ref()
    nl, nr = len(lkeys[0]), len(rkeys[0])
    _chk(lib.refh_frame_merge(C.c_uint64(nl), C.c_uint64(nr), len(lkeys), dts, la, ra, jobs, C.byref(m), None, None))
    li = np.empty(max(1, m.value), np.uint64)
    ri = np.empty(max(1, m.value), np.uint64)
    _chk(lib.refh_frame_merge(C.c_uint64(nl), C.c_uint64(nr), len(lkeys), dts, la, ra, jobs, C.byref(m),
                              C.c_void_p(li.ctypes.data), C.c_void_p(ri.ctypes.data)))
    return li[:m.value], ri[:m.value]


def ref_frame_vec(op: str, a, b=None, scalar: float = 0.0, cmp: str = "lt", jobs: int = 1):
    a = np.ascontiguousarray(a, np.float64)
    code = {"vector_add": 0, "multiply": 1, "scalar_compare": 2, "cumsum": 3, "reduce_sum": 4}[op]
    out = np.empty(max(1, len(a)), np.int64 if op == "scalar_compare" else np.float64)
    bb = np.ascontiguousarray(b if b is not None else a, np.float64)
    lib = ref()
    lib.refh_frame_vec.argtypes = [C.c_int, C.c_uint64, C.c_void_p, C.c_void_p, C.c_double, C.c_int, C.c_uint,
                                   C.c_void_p]
    _chk(lib.refh_frame_vec(code, len(a), a.ctypes.data, bb.ctypes.data, scalar, FRAME_OPS[cmp], jobs,
                            out.ctypes.data))
    return out[0] if op == "reduce_sum" else out[:len(a)]


# CPU restatement (test infrastructure), pinned to the reference by tests/test_oracle.py
def frame_key(col: np.ndarray, descending: bool = False) -> np.ndarray:
    """Order-preserving u64 key (frame.cpp:19-25: NaN above every number and
    equal to itself; -0 == +0)."""
    if col.dtype == np.int64:
        k = col.view(np.uint64) ^ np.uint64(1 << 63)
    elif col.dtype == np.uint64:
        k = col.copy()
    else:
        v = np.where(col == 0.0, 0.0, col)
        b = v.view(np.uint64)
        k = np.where(b >> np.uint64(63), ~b, b | np.uint64(1 << 63))
        k = np.where(np.isnan(col), np.uint64(~np.uint64(0)), k)
    return ~k if descending else k


def frame_argsort(keys, ascending=None) -> np.ndarray:
    ks = [frame_key(k, ascending is not None and not ascending[i]) for i, k in enumerate(keys)]
    return np.lexsort(ks[::-1]).astype(np.uint64)  # stable; keys[0] most significant


def frame_block_scan(a: np.ndarray):
    """reduce_sum and cumulative_sum (frame.cpp:599-647): fold left inside
    4096-element blocks, then across the block sums."""
    a = np.asarray(a, np.float64)
    out = np.empty_like(a)
    blocks = [a[i:i + 4096] for i in range(0, len(a), 4096)]
    sums = [np.cumsum(b)[-1] for b in blocks]
    carry = 0.0
    total = 0.0
    for i, b in enumerate(blocks):
        run = np.cumsum(b)
        out[i * 4096:i * 4096 + len(b)] = run if i == 0 else carry + run
        total = sums[0] if i == 0 else total + sums[i]
        carry = total
    return (total if len(a) else 0.0), out

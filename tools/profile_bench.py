"""Profile-record path at C4 scale (aurora-like, 1,000 nodes x 100 ranks):
device time of psg_slice (all rank profiles, the call sites + root, cputime
inclusive) and psg_profile_outliers, against the reference's ingest_profiles
and congestion_report on the host cores (oracle/_ref)."""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2605_03561_b200 import Context, scenarios  # noqa: E402

rpn = int(sys.argv[1]) if len(sys.argv) > 1 else 100
d = tempfile.mkdtemp()
truth = oracle.ref_generate(scenarios.aurora(ranks_per_node=rpn, seed=42), d)
meta = oracle.read_meta(d)
metric = next(m for (m, sc, n) in meta["metrics"] if n == "cputime" and sc == 1)
sites = truth["callsite_ctx"]
rank_pids = [p for (p, r, _) in meta["profiles"] if r >= 0]
ctxs = sorted([0] + list(sites))
out = {"ranks": len(rank_pids), "sites": len(sites)}
with Context(0) as ctx:
    ctx.load_profile_db(d)
    for _ in range(3):
        s = ctx.slice(rank_pids, ctxs, [metric])
        ctx.profile_outliers(metric, sites, top_k=0, z_min=1.0)
    t = []
    for _ in range(10):
        a = time.perf_counter()
        s = ctx.slice(rank_pids, ctxs, [metric])
        t.append(time.perf_counter() - a)
    out["gpu_slice_ms"] = 1e3 * float(np.median(t))
    out["slice_rows"] = int(len(s["pid"]))
    ms = [ctx.profile_outliers(metric, sites, top_k=0, z_min=1.0)["ms_total"] for _ in range(10)]
    out["gpu_profile_outliers_ms_device"] = float(np.median(ms))
    out["n_outliers"] = ctx.info["n_outliers"]
    # parity with the reference's congestion_report at this size
    rep = json.loads(oracle.ref_congestion_report(d))
    hosts = sorted({h for (_, r, h) in meta["profiles"] if r >= 0})
    o = ctx.outliers(len(hosts))
    want = [s["balance_ratio"] for s in rep["callsites"]]
    out["parity"] = {
        "worst_site": ctx.info["worst_site"] == rep["worst"]["ctx_id"],
        "balance_ratio_max_rel_err": float(np.max(np.abs(o["site_ratio"] - want) / np.abs(want))),
        "outliers_equal_dbscan_group": sorted(hosts[i] for i in o["selected"]) == sorted(rep["outlier_group"]["hostnames"]),
        "racks": [int(r[0]) for r in o["racks"]] == [r["rack"] for r in rep["topology"]["racks"]],
    }
lib = oracle.ref()
lib.refh_time_slices.restype = C.c_double
lib.refh_time_slices.argtypes = [C.c_char_p, C.POINTER(C.c_uint32), C.c_uint32, C.c_uint16, C.c_uint, C.c_uint]
cx = np.array(ctxs, np.uint32)
jobs = os.cpu_count()
out["cpu_cores"] = jobs
out["cpu_ingest_profiles_ms"] = 1e3 * lib.refh_time_slices(d.encode(), cx.ctypes.data_as(C.POINTER(C.c_uint32)),
                                                           len(cx), metric, jobs, 5)
out["cpu_congestion_report_ms"] = 1e3 * lib.refh_time_congestion(d.encode(), jobs, 2)
print(json.dumps(out))

"""configs[2] (C3) at full size: 8,192 ranks x 500 iterations x 64 kernels,
GAMESS-like spread (274 M events).  The UNMODIFIED reference generator writes
the database; the reference's build_tri_model + savings_report +
iteration_cv_report run on all host cores (oracle/_ref) and the GPU query
(cube + statistics) runs from the same trace.db; the cube, iteration counts,
gap rows and block offsets must be bit-identical and the diagnostics within
1e-9.  Prints one JSON line with both timings."""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2605_03561_b200 import Q_CUBE, Q_STATS, Context, scenarios  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
d = tempfile.mkdtemp(dir="/dev/shm" if os.path.isdir("/dev/shm") else None)
t = time.perf_counter()
oracle.ref_generate(scenarios.c3(n), d)
res = {"ranks": n, "gen_s": round(time.perf_counter() - t, 1)}
jobs = os.cpu_count()
t = time.perf_counter()
ref = oracle.ref_trimodel(d, 1, jobs=jobs, total_time=100.0)
res["cpu_trimodel_stats_s"] = round(time.perf_counter() - t, 2)
res["cpu_cores"] = jobs
with Context(0) as ctx:
    ctx.load_trace_db(d)
    res["events"] = int(ctx.shard()["n_events"])
    for _ in range(2):
        info = ctx.query(Q_CUBE | Q_STATS, anchor=1)
    ms = [ctx.query(Q_CUBE | Q_STATS, anchor=1)["ms_total"] for _ in range(5)]
    res["gpu_query_ms"] = round(float(np.median(ms)), 3)
    res["events_per_s_gpu"] = res["events"] / (res["gpu_query_ms"] / 1e3)
    res["events_per_s_cpu"] = res["events"] / res["cpu_trimodel_stats_s"]
    g = ctx.cube()
    ok = {k: bool(np.array_equal(g[k], ref[k])) for k in ("node_ids", "incl", "excl", "gap_incl", "gap_excl",
                                                           "block_offset")}
    ok["iter_counts"] = bool(np.array_equal(g["iter_counts"][g["iter_counts"] > 0], ref["iter_counts"]))
    s = ctx.stats(float(ref["savings_summary"][2]))
    rel = lambda a, b: float(np.max(np.abs(np.asarray(a) - np.asarray(b)) / np.maximum(np.abs(b), 1e-300)))  # noqa: E731
    res["savings_max_rel_err"] = rel(s["savings"].ravel(), ref["savings"])
    cv_ok = ref["cv_ok"].astype(bool)
    res["cv_max_rel_err"] = rel(s["cv"][cv_ok].ravel(), ref["cv"].reshape(-1, 2)[cv_ok].ravel())
    res["bit_exact"] = ok
    res["cells"] = int(info["n_cells"])
print(json.dumps(res))

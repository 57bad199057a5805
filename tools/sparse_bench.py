"""Throughput of the sparse window path (large calling-context trees): a
100,000-context tree (AMG-like), N traces x E events with
contexts drawn over the whole tree; window [T/4, 3T/4) group_aggregate +
rematerialize rows, and the cube of a small anchor subtree (global column
table).  Prints one JSON line (events/s, device ms per query)."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2605_03561_b200 import Q_CUBE, Q_WINDOW, Context  # noqa: E402

n_tr = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
n_ev = int(sys.argv[2]) if len(sys.argv) > 2 else 50_000
n_ctx = 100_000
rng = np.random.default_rng(1)
parent = np.empty(n_ctx, np.uint32)
parent[0] = 0xFFFFFFFF
parent[1:] = (rng.random(n_ctx - 1) * np.arange(1, n_ctx) ** 0.9).astype(np.uint32)
E = n_tr * n_ev
steps = rng.integers(0, 60, E).astype(np.uint64)
ts = np.cumsum(steps.reshape(n_tr, n_ev), axis=1).astype(np.uint64).ravel()
ctx = rng.integers(0, n_ctx, E).astype(np.uint32)
body = np.empty((E, 12), np.uint8)
body[:, :8] = ts.view(np.uint8).reshape(E, 8)
body[:, 8:] = ctx.view(np.uint8).reshape(E, 4)
off = np.arange(n_tr + 1, dtype=np.uint64) * n_ev
tend = ts.reshape(n_tr, n_ev)[:, -1] + 5
c = Context(0)
c.set_cct(parent)
c.load_aos(body.ravel(), off, np.arange(1, n_tr + 1, dtype=np.uint32), tend)
T = int(tend.max())
size = np.ones(n_ctx, np.int64)
for i in range(n_ctx - 1, 0, -1):
    size[parent[i]] += size[i]
anchor = int(np.flatnonzero((size >= 20) & (size <= 200))[0])
res = {}
for name, fl in (("window_sparse", Q_WINDOW), ("cube_global_cols", Q_CUBE)):
    ms, wall = [], []
    for i in range(int(os.environ.get("SPARSE_REPS", "12"))):
        t = time.perf_counter()
        info = c.query(fl, t0=T // 4, t1=3 * T // 4, anchor=anchor)
        wall.append(time.perf_counter() - t)
        ms.append(info["ms_total"])
    res[name] = {"ms_device": statistics.median(ms[4:]), "s_wall": statistics.median(wall[4:]), "ms_each": [round(x, 2) for x in ms],
                 "events_per_s_device": E / (statistics.median(ms[4:]) / 1e3),
                 "events_per_s_wall": E / statistics.median(wall[4:]),
                 "note": "median of queries 5..N (the first queries grow the output buffers)"}
    if fl == Q_WINDOW:
        res[name].update(rows=info["n_window_rows"], groups=info["n_window_groups"], remat=info["n_remat_rows"])
print(json.dumps({"traces": n_tr, "events_per_trace": n_ev, "events": E, "n_ctx": n_ctx, "anchor_subtree": int(size[anchor]),
                  **res}))

"""Times k_trace_query per query flavour (window only / cube only / cube+stats /
full) on a configs[1]-shaped shard: where does the fused kernel's time go?"""
import json
import statistics
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2605_03561_b200 import Q_CUBE, Q_EXACT_BOUNDS, Q_NO_CUBE_STORE, Q_STATS, Q_WINDOW, Context, scenarios  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
only = sys.argv[2] if len(sys.argv) > 2 else None  # run one flavour (for ncu)
ctx = Context(0)
ctx.generate_iterative(scenarios.device_scenario(n, 746, seed=1))
T = ctx.shard()["t_max"]
ev = ctx.shard()["n_events"]
res = {}
for name, fl in [("window", Q_WINDOW), ("cube", Q_CUBE), ("cube_nostore", Q_CUBE | Q_NO_CUBE_STORE),
                 ("cube_stats", Q_CUBE | Q_STATS), ("window_cube", Q_WINDOW | Q_CUBE),
                 ("full", Q_WINDOW | Q_CUBE | Q_STATS),
                 ("full_exact", Q_WINDOW | Q_CUBE | Q_STATS | Q_EXACT_BOUNDS)]:
    if only and name != only:
        continue
    ms, mb, mt = [], [], []
    for i in range(6):
        info = ctx.query(fl, t0=T // 4, t1=3 * T // 4, anchor=1)
        if i >= 2:
            ms.append(info["ms_main"])
            mb.append(info["ms_bounds"])
            mt.append(info["ms_total"])
    res[name] = {"ms": statistics.mean(ms), "bounds_ms": statistics.mean(mb),
                 "total_ms": statistics.mean(mt), "Gev_s": ev / statistics.mean(ms) / 1e6}
print(json.dumps({"traces": n, "events": ev, "k_trace_query": res}))

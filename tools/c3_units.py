"""configs[2] (C3) shape on the device generator: 8,192 GAMESS-like ranks x 500
iterations x 64 kernels (274 M events), cube + statistics query, with the
default work-unit plan (long traces split across warps) and with one warp per
trace (PSG_UNIT_EVENTS = 2^40); per-kernel times.  Prints one JSON line."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_03561_b200 import Q_ALL, Q_CUBE, Q_STATS, Context, scenarios  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
res = {"ranks": n}
with Context(0) as ctx:
    ctx.generate_iterative(scenarios.device_scenario(n, 500, spread="gamess", seed=3))
    sh = ctx.shard()
    res["events"] = int(sh["n_events"])
    T = int(sh["t_max"])
    for name, env in (("units", None), ("one_warp_per_trace", str(1 << 40))):
        if env:
            os.environ["PSG_UNIT_EVENTS"] = env
        else:
            os.environ.pop("PSG_UNIT_EVENTS", None)
        for flav, fl in (("cube_stats", Q_CUBE | Q_STATS), ("full", Q_ALL & ~(1 << 3))):
            kw = dict(t0=T // 4, t1=3 * T // 4, anchor=1) if flav == "full" else dict(anchor=1)
            for _ in range(3):
                ctx.query(fl, **kw)
            infos = [ctx.query(fl, **kw) for _ in range(10)]
            r = {k: round(statistics.median(i[k] for i in infos), 4) for k in ("ms_total", "ms_main", "ms_bounds")}
            r["events_per_s"] = res["events"] / (r["ms_total"] / 1e3)
            r["cube_store_bytes"] = infos[-1]["cube_store_bytes"]
            res[f"{name}/{flav}"] = r
print(json.dumps(res))

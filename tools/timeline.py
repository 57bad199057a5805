"""Per-query device time (ms_total, first to last event of psg_query) against
wall time and the stream-event time around back-to-back queries, per flag set,
at configs[1] scale: where does the step time go outside the kernels?"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_03561_b200 import Q_ALL, Q_CUBE, Q_STATS, Q_WINDOW, Context, scenarios  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = Context(0, stream=stream.cuda_stream)
ctx.generate_iterative(scenarios.device_scenario(n, 746, seed=1))
sh = ctx.shard()
T = sh["t_max"]
node_of = (np.arange(n) // 100).astype(np.uint32)
nn_ = (n + 99) // 100
node = np.arange(nn_)
ctx.set_nodes(node_of, nn_, 4000 + node // 32, (node // 8) % 4)
out = {}
for name, fl in [("all", Q_ALL), ("no_outliers", Q_WINDOW | Q_CUBE | Q_STATS)]:
    q = dict(flags=fl, t0=T // 4, t1=3 * T // 4, anchor=1, sites=list(range(2, 66)) if fl == Q_ALL else (),
             top_k=32 if fl == Q_ALL else 0, z_min=float("-inf"))
    for _ in range(2):
        ctx.query(**q)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tot, walls = [], []
    e0.record(stream)
    for _ in range(4):
        w0 = time.perf_counter()
        info = ctx.query(**q)
        walls.append((time.perf_counter() - w0) * 1e3)
        tot.append(info["ms_total"])
    e1.record(stream)
    torch.cuda.synchronize()
    out[name] = {"stream_ms_per_query": e0.elapsed_time(e1) / 4, "ms_total": float(np.mean(tot)),
                 "wall_ms": float(np.mean(walls)), "ms_main": info["ms_main"], "ms_bounds": info["ms_bounds"]}
print(json.dumps(out))

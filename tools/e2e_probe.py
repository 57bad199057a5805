"""Breakdown of bench.py's e2e step at configs[1] (one GPU): the trace load
alone (pinned host trace.db bytes -> HBM SoA), the query, the window / stats /
outlier copy-out, the cube's stored-form copy-out alone, and the overlapped
step.  Prints one JSON line; measurement plumbing, not product."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2605_03561_b200 import Q_ALL, Context, scenarios  # noqa: E402

n, iters = 100_000, 746
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = Context(0, stream=stream.cuda_stream)
ctx.generate_iterative(scenarios.device_scenario(n, iters, seed=1), 0, n)
sh = ctx.shard()
node_of = (np.arange(n) // 100).astype(np.uint32)
nodes = (n + 99) // 100
node = np.arange(nodes)
ctx.set_nodes(node_of, nodes, 4000 + node // 32, (node // 8) % 4)
T = sh["t_max"]
q = dict(flags=Q_ALL, t0=T // 4, t1=3 * T // 4, anchor=1, sites=list(range(2, 66)), top_k=32,
         z_min=float("-inf"))
info = ctx.query(**q)
host = torch.empty(sh["n_events"] * 12, dtype=torch.uint8, pin_memory=True)
ctx.export_aos(host.data_ptr())
idx = ctx.index()
off, pids, tend = idx["off"], idx["pid"], idx["t_end"]
cube_pin = (torch.empty(info["cube_store_bytes"] + 16, dtype=torch.uint8, pin_memory=True),
            torch.empty(8 * (info["n_cells"] // max(1, info["n_nodes"])) * info["n_internal"] + 8,
                        dtype=torch.uint8, pin_memory=True))
cube_np = (cube_pin[0].numpy().view(np.uint32 if info["cube_cell_bytes"] == 4 else np.uint64),
           cube_pin[1].numpy().view(np.int64))
off_pin = torch.empty(8 * n + 8, dtype=torch.uint8, pin_memory=True).numpy().view(np.uint64)


def timed(f, reps=3):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        f()
        torch.cuda.synchronize()
        out.append(time.perf_counter() - t)
    return min(out)


def load():
    ctx.load_aos(host.data_ptr(), off, pids, tend)
    ctx.set_nodes(node_of, nodes, 4000 + node // 32, (node // 8) % 4)


r = {}
r["load_s"] = timed(load)
r["load_gbs"] = sh["n_events"] * 12 / r["load_s"] / 1e9
r["query_s"] = timed(lambda: ctx.query(**q))
r["window_stats_outliers_s"] = timed(lambda: (ctx.window(), ctx.stats(1.0), ctx.outliers(nodes),
                                               ctx.cube(with_cells=False)))
r["cube_stored_sync_s"] = timed(lambda: ctx.cube_stored(*cube_np, wait=True, off_out=off_pin))
r["cube_bytes"] = int(cube_np[0].nbytes + cube_np[1].nbytes)
r["cube_gbs"] = r["cube_bytes"] / r["cube_stored_sync_s"] / 1e9


def load_during_cube():
    ctx.cube_stored(*cube_np, wait=False, off_out=off_pin)
    load()
    ctx.query(**q)
    ctx.wait_copies()


r["cube_then_load_overlapped_s"] = timed(load_during_cube)
print(json.dumps(r))

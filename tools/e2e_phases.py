"""Per-phase host timings of bench.py's e2e step at configs[1] in the steady
state (the cube's async copy-out overlapping the next load), so the gap to
the PCIe bound can be attributed.  Measurement plumbing, not product."""
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
pin = {k: torch.empty(n * sh["n_ctx"] * 8, dtype=torch.uint8, pin_memory=True) for k, _ in Context.WINDOW_DTYPES}
wout = {k: pin[k].numpy().view(dt).reshape(n, sh["n_ctx"]) for k, dt in Context.WINDOW_DTYPES}
cube_pin = (torch.empty(info["cube_store_bytes"] + 16, dtype=torch.uint8, pin_memory=True),
            torch.empty(8 * (info["n_cells"] // max(1, info["n_nodes"])) * info["n_internal"] + 8,
                        dtype=torch.uint8, pin_memory=True))
cube_np = (cube_pin[0].numpy().view(np.uint32 if info["cube_cell_bytes"] == 4 else np.uint64),
           cube_pin[1].numpy().view(np.int64))
off_pin = torch.empty(8 * n + 8, dtype=torch.uint8, pin_memory=True).numpy().view(np.uint64)
phases = {}


def step():
    t = [time.perf_counter()]
    ctx.load_aos(host.data_ptr(), off, pids, tend); t.append(time.perf_counter())
    ctx.set_nodes(node_of, nodes, 4000 + node // 32, (node // 8) % 4); t.append(time.perf_counter())
    ctx.query(**q); t.append(time.perf_counter())
    ctx.window(wout); t.append(time.perf_counter())
    ctx.stats(1.0); t.append(time.perf_counter())
    ctx.outliers(nodes); t.append(time.perf_counter())
    ctx.cube(with_cells=False); t.append(time.perf_counter())
    ctx.cube_stored(*cube_np, wait=False, off_out=off_pin); t.append(time.perf_counter())
    for name, a, b in zip(("load", "set_nodes", "query", "window", "stats", "outliers", "cube_meta",
                           "cube_async_launch"), t, t[1:]):
        phases.setdefault(name, []).append(b - a)


step()
ctx.wait_copies()
phases.clear()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(6):
    step()
ctx.wait_copies()
torch.cuda.synchronize()
tot = (time.perf_counter() - t0) / 6
print(json.dumps({"s_per_step": tot, **{k: float(np.median(v)) for k, v in phases.items()}}))

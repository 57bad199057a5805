"""The paper's Query API op set (Tables 1-3: grouping, sorting,
filtering, merging; vector add, in-place multiply, scalar compare, reduction
sum, cumulative sum) on trace-shaped tables: the GPU frame operators
(device-resident columns, CUDA events) against the reference's frame engine
on all host cores (oracle/_ref).  Rows = traces x events per trace."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2605_03561_b200 import Context, frame  # noqa: E402

traces = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
per = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
n = traces * per
rng = np.random.default_rng(7)
k0 = np.repeat(np.arange(traces, dtype=np.uint64), per)                 # profile id
k1 = rng.integers(0, 67, n).astype(np.uint64)                         # ctx id
k2 = np.cumsum(rng.integers(1, 1000, n)).astype(np.uint64)             # timestamp
v = rng.random(n)                                                     # duration (s)
mk = np.arange(traces, dtype=np.uint64)
mv = rng.random(traces)
res = {"traces": traces, "rows": n}
ctx = Context(0)
t = frame.Table(ctx)
for name, arr in (("k0", k0), ("k1", k1), ("k2", k2), ("v", v)):
    t.add_column(frame.Column.from_numpy(name, arr))
r = frame.Table(ctx)
r.add_column(frame.Column.from_numpy("k0", mk))
r.add_column(frame.Column.from_numpy("w", mv))
lit = int(k2[n // 2])
V = t.col("v")
ops = {
    "grouping": lambda: frame.group_aggregate(t, ["k0", "k1"], [("v", f) for f in ("sum", "min", "max", "mean", "count")]),
    "sorting": lambda: frame.sort(t, ["k0", "k2"], [True, False]),
    "filtering": lambda: frame.filter(t, "k2", "ge", lit),
    "merging": lambda: frame.merge(t, r, ["k0"]),
    "vector_add": lambda: frame.vector_add(ctx, V, V),
    "in_place_multiply": lambda: frame.in_place_multiply(ctx, V, 1.5),
    "scalar_compare": lambda: frame.scalar_compare(ctx, V, "gt", 0.5),
    "reduce_sum": lambda: frame.reduce_sum(ctx, V),
    "cumulative_sum": lambda: frame.cumulative_sum(ctx, V),
}
lib = oracle.ref()
lib.refh_time_frame.restype = C.c_double
P = C.c_void_p
lib.refh_time_frame.argtypes = [C.c_int, C.c_uint64, P, P, P, P, C.c_uint64, P, P, C.c_uint64, C.c_uint, C.c_uint]
jobs = os.cpu_count()
for code, (name, fn) in enumerate(ops.items()):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        fn()
    e1.record()
    torch.cuda.synchronize()
    gpu_ms = e0.elapsed_time(e1) / 5
    cpu_ms = 1e3 * lib.refh_time_frame(code, n, k0.ctypes.data, k1.ctypes.data, k2.ctypes.data, v.ctypes.data,
                                       traces, mk.ctypes.data, mv.ctypes.data, lit, jobs, 2)
    res[name] = {"gpu_ms": round(gpu_ms, 4), "cpu_ms": round(cpu_ms, 3), "speedup": round(cpu_ms / gpu_ms, 1)}
res["cpu_cores"] = jobs
print(json.dumps(res))

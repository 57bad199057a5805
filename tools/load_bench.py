"""Storage -> HBM ingest: writes a configs[1]-shaped
trace database (meta.bin + trace.db in the reference format) to a directory,
then times psg_load_trace_db from it (the mmap'd, page-cache-resident file
goes through the pinned staging ring) next to psg_load_traces_aos from pinned
host memory.  Prints one JSON line."""
from __future__ import annotations

import json
import os
import struct
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_03561_b200 import Context, scenarios  # noqa: E402


def put_str(s: str) -> bytes:
    b = s.encode()
    return struct.pack("<H", len(b)) + b


def write_db(ctx: Context, d: str, parent) -> int:
    os.makedirs(d, exist_ok=True)
    idx = ctx.index()
    n = len(idx["pid"])
    meta = b"HPAN" + struct.pack("<I", 1)
    meta += struct.pack("<I", 1) + struct.pack("<IB", 0, 0) + put_str("cputime") + put_str("s")
    meta += struct.pack("<I", n)
    for i, p in enumerate(idx["pid"]):
        meta += struct.pack("<Iii", int(p), i, 0) + put_str(f"x1000c0s0b0n{i // 100}") + struct.pack("<Q", 0)
    meta += struct.pack("<I", len(parent))
    for c, par in enumerate(parent):
        meta += struct.pack("<IIB", c, int(par), 0) + put_str(f"c{c}")
    open(os.path.join(d, "meta.bin"), "wb").write(meta)
    body = torch.empty(int(idx["off"][-1]) * 12, dtype=torch.uint8, pin_memory=True)
    ctx.export_aos(body.data_ptr())
    with open(os.path.join(d, "trace.db"), "wb") as f:
        f.write(b"HPTR" + struct.pack("<II", 1, n))
        base = 12 + 36 * n
        tb = body.numpy()
        for t in range(n):
            cnt = int(idx["off"][t + 1] - idx["off"][t])
            o = base + 12 * int(idx["off"][t])
            t0 = int(tb[12 * int(idx["off"][t]):12 * int(idx["off"][t]) + 8].view(np.uint64)[0]) if cnt else 0
            f.write(struct.pack("<IQQQQ", int(idx["pid"][t]), o, cnt, t0, int(idx["t_end"][t])))
        f.write(tb.tobytes())
    return body.numel()


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
    d = sys.argv[2] if len(sys.argv) > 2 else "/dev/shm/psg_load_bench"
    ctx = Context(0)
    ctx.generate_iterative(scenarios.device_scenario(n, 746, seed=1))
    parent = np.array([0xFFFFFFFF, 0] + [1] * 64 + [0], np.uint32)
    nbytes = write_db(ctx, d, parent)
    idx = ctx.index()
    res = {"traces": n, "bytes": nbytes}
    for name, fn in [("trace_db_mmap", lambda: ctx.load_trace_db(d))]:
        fn()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        res[name + "_GBps"] = 3 * nbytes / (time.perf_counter() - t) / 1e9
    pinned = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    with open(os.path.join(d, "trace.db"), "rb") as f:
        f.seek(12 + 36 * n)
        pinned.numpy()[:] = np.frombuffer(f.read(), np.uint8)
    ctx.set_cct(parent)
    t = time.perf_counter()
    for _ in range(3):
        ctx.load_aos(pinned.data_ptr(), idx["off"], idx["pid"], idx["t_end"])
    torch.cuda.synchronize()
    res["pinned_aos_GBps"] = 3 * nbytes / (time.perf_counter() - t) / 1e9
    print(json.dumps(res))


if __name__ == "__main__":
    main()

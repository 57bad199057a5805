#!/usr/bin/env python
"""Benchmark of BASELINE.json's metric: trace events/s of the full trace query
(window filter + per-(trace,ctx) aggregates + iteration cube + cross-rank
stats + outlier top-k) over configs[1] = 100,000 synthetic traces x 49,982
events (5.0e9 events), sharded by rank over N GPUs (one process per GPU).

  python bench.py [--gpus N --steps K --warmup W]          # our arm
  python bench.py --impl reference [...]                   # the reference's CPU path

One JSON line is printed by rank 0.  See DESIGN.md §Measurement for every key.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "trace events/s over 100k synthetic traces at 1/2/4/8 B200; x vs CPU ref"
N_TRACES = 100_000
N_ITERS = 746
EVENTS_PER_TRACE = N_ITERS * 67
CPU_SAMPLE_TRACES = 400  # ranks 0..399 of configs[1]: 20.0M events, ~10-30 s of host work


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--traces", type=int, default=N_TRACES)
    ap.add_argument("--iters", type=int, default=N_ITERS)
    ap.add_argument("--e2e-steps", type=int, default=12)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--prefetch", action="store_true",
                    help="e2e with psg_prefetch_aos (A/B: neutral, profiles/r2o_ab_e2e_prefetch.txt)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=CPU_SAMPLE_TRACES)
    return ap.parse_args()


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 50 ms while active."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(self.rows[0][1]) if self.rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(self.rows)}


def measured_peak() -> tuple[float, str]:
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_kernels() -> dict:
    """Per-event DRAM bytes (read + write) of the query's big kernels, from the
    committed ncu capture at configs[1] (profiles/ncu_summary.json)."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        d = json.load(open(p))
        return {k: (v["dram_bytes_read"] + v["dram_bytes_write"]) / d["events"]
                for k, v in d["kernels"].items()} | {"_source": d["round"]}
    except Exception:
        return {}


# ---------------------------------------------------------------------------
def cpu_reference_sample(n_sample: int, repeat: int) -> dict:
    """The reference's own CPU query (oracle/_ref: ingest_traces + group_aggregate
    + build_tri_model + savings/CV) on ranks 0..n_sample-1 of configs[1]."""
    import oracle
    from paper_2605_03561_b200 import scenarios
    base = "/dev/shm" if os.path.isdir("/dev/shm") else tempfile.gettempdir()
    cfg = scenarios.c2(n_ranks=n_sample)
    with tempfile.TemporaryDirectory(dir=base) as d:
        oracle.ref_generate(cfg, d)
        tr = oracle.read_trace_db(d)
        T = int(tr["t_end"].max())
        events = int(tr["off"][-1])
        jobs = int(oracle.ref().refh_default_jobs())
        secs = [oracle.ref().refh_time_query(d.encode(), T // 4, 3 * T // 4, 1, jobs, 1)
                for _ in range(repeat)]
    if min(secs) < 0:
        raise RuntimeError(oracle.ref().refh_last_error().decode())
    return {"events": events, "secs": secs, "cores": jobs,
            "sample": f"ranks 0..{n_sample - 1} of configs[1] ({n_sample} traces x {EVENTS_PER_TRACE} "
                      f"events = {events} events), window [T/4,3T/4), anchor ctx 1; reference "
                      f"ingest_traces+group_aggregate+build_tri_model+savings_report+"
                      f"iteration_cv_report, jobs={jobs}"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    s = cpu_reference_sample(args.cpu_sample, args.warmup + args.steps)
    timed = s["secs"][args.warmup:] or s["secs"]
    v = s["events"] / statistics.mean(timed)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "events/s",
        "n_gpus": args.gpus, "steps": len(timed), "warmup": args.warmup,
        "ms_per_step": 1000 * statistics.mean(timed), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": f"configs[1] sample: {s['sample']}", "traces": args.cpu_sample,
                   "events_per_trace": EVENTS_PER_TRACE},
        "cpu_baseline": {"value": v, "unit": "events/s", "cores": s["cores"], "kind": "reference",
                         "sample": s["sample"]},
        "e2e": {"value": v, "unit": "events/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2605_03561_b200 import Q_ALL, Context, scenarios

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)

    n = args.traces
    # shards: contiguous rank ranges balanced by events with edges on node
    # boundaries (100 ranks per node), so node means stay shard-local
    # (every trace of this workload has the same length)
    from paper_2605_03561_b200 import dist as pdist
    lo, hi = pdist.node_aligned_ranges(np.arange(n) // 100, world,
                                       np.full(n, args.iters * 67, np.float64))[rank]
    ctx = Context(local, stream=stream.cuda_stream)
    if world > 1:
        uid = [Context.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.comm_init(world, rank, uid[0])

    cfg = scenarios.device_scenario(n, args.iters, seed=1)
    ctx.generate_iterative(cfg, lo, hi)
    sh = ctx.shard()
    n_local, events_local = sh["n_traces"], sh["n_events"]
    # rank -> node: 100 ranks per node (C4's aurora shape), 4 chassis x 8 slots per rack
    node_of = (np.arange(lo, hi) // 100).astype(np.uint32)
    n_nodes = (n + 99) // 100
    node = np.arange(n_nodes)
    ctx.set_nodes(node_of, n_nodes, 4000 + node // 32, (node // 8) % 4)
    tmax = torch.tensor([sh["t_max"]], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    T = int(tmax.item())
    q = dict(flags=Q_ALL, t0=T // 4, t1=3 * T // 4, anchor=1, sites=list(range(2, 66)),
             top_k=32, z_min=float("-inf"))

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        ctx.query(**q)
    torch.cuda.synchronize()
    info = ctx.info
    launches0 = Context.kernel_launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    main_ms, bounds_ms = [], []
    with ClockSampler(local) as clocks:
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            info = ctx.query(**q)
            main_ms.append(info["ms_main"])
            bounds_ms.append(info["ms_bounds"])
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    launches = (Context.kernel_launches() - launches0) // max(1, args.steps)
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    total_events = n * args.iters * 67
    value = total_events / (ms_max / 1000.0 / args.steps)

    # roofline of the dominant kernel (k_trace_query): algorithmic bytes per launch
    nn, n_ctx = info["n_nodes"], sh["n_ctx"]
    # algorithmic bytes of k_trace_query: events read once (12 B),
    # the compact cube written (incl as stored: 4 or 8 B per cell in rows of
    # nn + 1 rounded to even, + excl 8 B per internal node per iteration),
    # boundary windows read (4 + 8 B per iteration), window rows (7 x 8 B per
    # (trace, ctx)), gap rows (16 B per kept trace x node) and the within-rank
    # CV outputs (9 B per kept trace x node)
    rows = info["n_cells"] // max(1, nn)
    alg_bytes = (12 * events_local + info["cube_store_bytes"] + 8 * rows * info["n_internal"] + 12 * rows
                 + 56 * n_local * n_ctx + 16 * info["n_kept"] * nn + 9 * info["n_kept"] * nn)
    main_s = statistics.mean(main_ms) / 1000.0
    peak, peak_kind = measured_peak()
    achieved = alg_bytes / main_s / 1e9
    ncu = ncu_kernels()
    per_ev = ncu.get("k_trace_query")
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "peak_kind": peak_kind,
                # ncu dram__bytes_read + _write of this kernel at this config
                # (one launch, profiles/ncu_summary.json), scaled to this shard
                "traffic": per_ev * events_local if per_ev else None,
                "traffic_source": ncu.get("_source"),
                "kernel": "k_trace_query", "alg_bytes_per_launch": alg_bytes,
                "cube_cell_bytes": info["cube_cell_bytes"],
                "kernel_ms": main_s * 1000.0, "kernel_share_of_step": main_s * 1000.0 / (ms / args.steps),
                "pass1_k_bounds_ms": statistics.mean(bounds_ms),
                "frac_of_nominal_8tbs": achieved / 8000.0}
    # the whole query step: its algorithmic bytes are the
    # events read ONCE plus every output written once -- the same bytes as
    # k_trace_query's (the statistics and outlier outputs are < 1 MB).  The
    # DRAM traffic adds what the step re-reads: pass 1's 1-byte ctx mirror
    # (k_bounds) and the stored cube (k_cross_stats); wasted_traffic_ratio =
    # measured DRAM bytes of the three kernels / algorithmic bytes.
    step_s = ms / args.steps / 1000.0
    dram = (sum(ncu[k] for k in ("k_bounds", "k_trace_query", "k_cross_stats")) * events_local
            if all(k in ncu for k in ("k_bounds", "k_trace_query", "k_cross_stats")) else None)
    roofline["step"] = {"alg_bytes": alg_bytes, "achieved": alg_bytes / step_s / 1e9,
                        "frac": alg_bytes / step_s / 1e9 / peak,
                        "dram_bytes": dram, "wasted_traffic_ratio": dram / alg_bytes if dram else None,
                        "dram_frac": dram / step_s / 1e9 / peak if dram else None}

    # end to end through the public API: pinned host trace.db bytes -> HBM ->
    # query -> results back to host, every step.
    e2e = None
    if not args.no_e2e:
        host = torch.empty(events_local * 12, dtype=torch.uint8, pin_memory=True)
        ctx.export_aos(host.data_ptr())
        idx = ctx.index()
        off, pids, tend = idx["off"], idx["pid"], idx["t_end"]
        # pinned host buffers for the window copy-out (allocated once, reused)
        n_cells = n_local * sh["n_ctx"]
        pin = {k: torch.empty(n_cells * 8, dtype=torch.uint8, pin_memory=True)
               for k, _ in Context.WINDOW_DTYPES}
        wout = {k: pin[k].numpy().view(dt).reshape(n_local, sh["n_ctx"]) for k, dt in Context.WINDOW_DTYPES}
        # the cube (the query's largest output) comes back too, in its stored
        # lossless form (32-bit incl cells + the internal nodes' excl), into
        # pinned buffers sized from the warm-up query
        cube_pin = None
        try:
            xrows = info["n_cells"] // max(1, nn) * info["n_internal"]
            cube_pin = (torch.empty(info["cube_store_bytes"] + 16, dtype=torch.uint8, pin_memory=True),
                        torch.empty(8 * xrows + 8, dtype=torch.uint8, pin_memory=True))
            cube_np = (cube_pin[0].numpy().view(np.uint32 if info["cube_cell_bytes"] == 4 else np.uint64),
                       cube_pin[1].numpy().view(np.int64))
        except Exception as e:  # host RAM too small to pin it: say so in the line
            cube_pin, cube_err = None, f"{type(e).__name__}: {e}"
        off_pin = torch.empty(8 * n_local + 8, dtype=torch.uint8, pin_memory=True).numpy().view(np.uint64)
        # pinned buffers for the cube's dense per-trace outputs (iteration
        # counts, block offsets, gap rows: ~0.1 GB at configs[1])
        cmeta = {"iter_counts": torch.empty(4 * n_local + 4, dtype=torch.uint8, pin_memory=True).numpy().view(np.uint32),
                 "block_offset": torch.empty(8 * n_local + 8, dtype=torch.uint8, pin_memory=True).numpy().view(np.uint64),
                 "gap_incl": torch.empty(8 * n_local * nn + 8, dtype=torch.uint8, pin_memory=True).numpy().view(np.int64),
                 "gap_excl": torch.empty(8 * n_local * nn + 8, dtype=torch.uint8, pin_memory=True).numpy().view(np.int64)}
        d2h = 0

        def e2e_step():
            # one step of the public API: this step's trace bytes in, every
            # result out.  The cube's copy-out is asynchronous: it lands while
            # the next step's traces stream in (PCIe is full duplex); the next
            # query waits for it on the device, and the clock stops only after
            # the last one landed (ctx.wait_copies below).
            ctx.load_aos(host.data_ptr(), off, pids, tend)
            ctx.set_nodes(node_of, n_nodes, 4000 + node // 32, (node // 8) % 4)
            # optionally the next step's first 1.5 GB of trace bytes cross PCIe
            # while this step's query and copy-out run (measured neutral)
            if args.prefetch:
                ctx.prefetch_aos(host.data_ptr(), events_local)
            ctx.query(**q)
            w = ctx.window(wout)
            st = ctx.stats(1.0)
            ou = ctx.outliers(n_nodes)
            cb = ctx.cube(with_cells=False, out=cmeta)
            cs = ctx.cube_stored(*cube_np, wait=False, off_out=off_pin) if cube_pin is not None else None
            return (sum(a.nbytes for a in w.values()) + sum(a.nbytes for a in st.values())
                    + sum(a.nbytes for a in ou.values())
                    + sum(a.nbytes for k, a in cb.items() if a is not None)
                    + (cs["incl"].nbytes + cs["xint"].nbytes + cs["stored_off"].nbytes if cs else 0))

        e2e_step()  # warms the staging buffers
        ctx.wait_copies()
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            d2h = e2e_step()
        ctx.wait_copies()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / args.e2e_steps
        tt = torch.tensor([dt], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        secs = [float(tt.item())]
        # the e2e roofline: PCIe.  Pinned H2D rate measured here on 4 GiB of the
        # same pinned buffer (one copy, CUDA events); the step cannot beat
        # h2d_bytes / that rate (the D2H runs on the other direction)
        hb = 4 << 30
        if host.numel() >= hb:
            dbuf = torch.empty(hb, dtype=torch.uint8, device="cuda")
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            dbuf.copy_(host[:hb], non_blocking=True)
            e1.record(stream)
            torch.cuda.synchronize()
            h2d_gbs = hb / (e0.elapsed_time(e1) / 1000.0) / 1e9
            del dbuf
        else:
            h2d_gbs = None
        h2d_b = int(events_local * 12 + 8 * (n_local + 1) + 12 * n_local)
        e2e_bound = {"bound": "pcie_h2d", "h2d_gbs": h2d_gbs,
                     "min_s_per_step": h2d_b / (h2d_gbs * 1e9) if h2d_gbs else None,
                     "frac": (h2d_b / (h2d_gbs * 1e9)) / statistics.mean(secs) if h2d_gbs else None}
        e2e = {"value": total_events / statistics.mean(secs), "unit": "events/s",
               "roofline": e2e_bound,
               "h2d_bytes_per_step": int(events_local * 12 + 8 * (n_local + 1) + 12 * n_local),
               "d2h_bytes_per_step": int(d2h), "steps": args.e2e_steps,
               "s_per_step": statistics.mean(secs),
               "note": "pinned trace.db bytes -> psg_load_traces_aos -> psg_query -> window/"
                       "stats/outliers/iteration counts and the cube (stored lossless form: "
                       "32-bit incl cells + internal-node excl, psg_get_cube_stored_async) copied "
                       "back into pinned host memory every step; the cube's D2H overlaps the next "
                       "step's H2D, the clock stops after the last one landed"
                       if cube_pin is not None else
                       "cube copy-out skipped: " + cube_err}
        del host

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            s = cpu_reference_sample(args.cpu_sample, 1)
            cpu = {"value": s["events"] / s["secs"][0], "unit": "events/s", "cores": s["cores"],
                   "kind": "reference", "sample": s["sample"]}
        except Exception as e:  # the reference build is missing on this box
            cpu = {"value": None, "unit": "events/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "events/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic (device replay of the reference generator, byte-identical)",
            "config": {"workload": f"configs[1]: {n} traces x {args.iters * 67} events "
                                   f"({total_events:.3e} events), full query: window [T/4,3T/4) "
                                   "filter+aggregate, iteration cube (anchor 1, materialised), "
                                   "savings/CV stats, 64-site outlier top-32 + topology",
                       "traces": n, "events": total_events, "parallelism": f"dp{world}",
                       "l2": "inputs (60 GB) >> L2 (126 MB); no flush needed"},
            "clocks": clocks.summary(), "gpu_launches": int(launches), "roofline": roofline,
            "e2e": e2e, "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

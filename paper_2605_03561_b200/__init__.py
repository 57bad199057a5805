"""perfslice-b200: the reference's trace query path (window filter, segmented
aggregates, iteration cube, z-score/top-k outliers) on hand-written sm_100a
kernels behind a C ABI (include/psg.h).

This module is the Python face of that ABI (ctypes); every computation runs
in libpsg.so on the GPU.  Importing it does not need a GPU; opening a Context
does, and fails loudly without one.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _lib
from ._lib import (ANCHOR_AUTO, PsgError, Q_ALL, Q_CLAMP_TEND, Q_CUBE, Q_CUBE64, Q_EXACT_BOUNDS, Q_NO_CUBE_STORE, Q_OUTLIERS, Q_SPARSE, Q_STATS, Q_WINDOW,
                   check, load)
from . import scenarios

__all__ = ["ANCHOR_AUTO", "Context", "PsgError", "Q_ALL", "Q_CLAMP_TEND", "Q_CUBE", "Q_CUBE64", "Q_EXACT_BOUNDS", "Q_NO_CUBE_STORE", "Q_OUTLIERS", "Q_SPARSE", "Q_STATS",
           "Q_WINDOW", "load", "scenarios"]


def _ptr(a: Optional[np.ndarray], ctype):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ctype))


class Context:
    """One psg_context: one GPU, one stream, one shard of traces."""

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        self.lib = load()
        h = C.c_void_p()
        check(self.lib.psg_open(device, C.c_void_p(stream) if stream else None, C.byref(h)))
        self.h = h
        self.info = None

    # -- lifetime ------------------------------------------------------------
    def close(self):
        if self.h:
            self.lib.psg_close(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return int(self.lib.psg_stream(self.h) or 0)

    # -- multi-GPU -----------------------------------------------------------
    @staticmethod
    def comm_unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(load().psg_comm_unique_id(buf))
        return bytes(buf)

    def comm_init(self, nranks: int, rank: int, uid: bytes):
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        check(self.lib.psg_comm_init(self.h, nranks, rank, buf))

    def comm_init_host(self, nranks: int, rank: int, reduce):
        """Summary exchange through a host reducer instead of NCCL:
        reduce(array, op) must reduce the numpy array (uint64 or float64) in
        place across ranks, op in {"sum", "max", "min"} (see dist.py)."""
        ops = ("sum", "max", "min")

        def cb(buf, count, dtype, op, _user):
            try:
                ctype = C.c_double if dtype == 1 else C.c_uint64
                arr = np.ctypeslib.as_array(C.cast(buf, C.POINTER(ctype)), shape=(count,))
                reduce(arr, ops[op])
                return 0
            except Exception:  # reported as PS_E_INTERNAL by the library
                return 1
        self._host_cb = _lib.ALLREDUCE_FN(cb)
        check(self.lib.psg_comm_init_host(self.h, nranks, rank, self._host_cb, None))

    # -- loading -------------------------------------------------------------
    def set_cct(self, parent):
        p = np.ascontiguousarray(parent, dtype=np.uint32)
        check(self.lib.psg_set_cct(self.h, _ptr(p, C.c_uint32), len(p)))

    def load_aos(self, body, event_off, profile_ids, t_end):
        """body: uint8 array (or an int host address) of packed 12-byte events."""
        off = np.ascontiguousarray(event_off, dtype=np.uint64)
        pid = np.ascontiguousarray(profile_ids, dtype=np.uint32)
        te = np.ascontiguousarray(t_end, dtype=np.uint64)
        n_ev = int(off[-1])
        addr = body if isinstance(body, int) else (body.ctypes.data if n_ev else 0)
        check(self.lib.psg_load_traces_aos(self.h, C.c_void_p(addr), n_ev, _ptr(off, C.c_uint64),
                                           _ptr(pid, C.c_uint32), _ptr(te, C.c_uint64), len(pid)))

    def prefetch_aos(self, body, n_events: int):
        """Start copying the first staging chunks of the next load_aos(body, ...)
        (same body, n_events events) while the device works on the current
        traces; pinned bodies only (else a no-op)."""
        addr = body if isinstance(body, int) else (body.ctypes.data if n_events else 0)
        check(self.lib.psg_prefetch_aos(self.h, C.c_void_p(addr), int(n_events)))

    def load_trace_db(self, path: str, pids=None):
        if pids is None:
            check(self.lib.psg_load_trace_db(self.h, path.encode(), None, 0))
        else:
            p = np.ascontiguousarray(pids, dtype=np.uint32)
            check(self.lib.psg_load_trace_db(self.h, path.encode(), _ptr(p, C.c_uint32), len(p)))

    def generate_iterative(self, cfg: dict, rank_lo: int = 0, rank_hi: Optional[int] = None):
        mean, jit, spread, stride = scenarios.device_params(cfg)
        s = _lib.IterScenario()
        s.n_ranks = cfg["n_ranks"]
        s.n_iterations = cfg["n_iterations"]
        s.n_kernels = len(mean)
        s.mean_time_s = _ptr(mean, C.c_double)
        s.jitter_frac = _ptr(jit, C.c_double)
        s.spread = _ptr(spread, C.c_double) if spread is not None else None
        s.spread_kernel_stride = stride
        s.copy_segment_s = cfg.get("copy_segment_s", 0.0)
        s.seed = cfg.get("seed", 0)
        self._keep = (mean, jit, spread)
        check(self.lib.psg_generate_iterative(self.h, C.byref(s), rank_lo,
                                              cfg["n_ranks"] if rank_hi is None else rank_hi))

    def set_nodes(self, node_of_trace, n_nodes, rack=None, chassis=None):
        nt = np.ascontiguousarray(node_of_trace, dtype=np.uint32)
        r = None if rack is None else np.ascontiguousarray(rack, dtype=np.uint32)
        c = None if chassis is None else np.ascontiguousarray(chassis, dtype=np.uint32)
        check(self.lib.psg_set_nodes(self.h, _ptr(nt, C.c_uint32), n_nodes, _ptr(r, C.c_uint32),
                                     _ptr(c, C.c_uint32)))

    def shard(self) -> dict:
        s = _lib.ShardInfo()
        check(self.lib.psg_shard(self.h, C.byref(s)))
        return {k: getattr(s, k) for k, _ in s._fields_}

    def traces(self):
        sh = self.shard()
        n, e = sh["n_traces"], sh["n_events"]
        ts = np.empty(e, np.uint64)
        cx = np.empty(e, np.uint32)
        off = np.empty(n + 1, np.uint64)
        te = np.empty(n, np.uint64)
        pid = np.empty(n, np.uint32)
        check(self.lib.psg_get_traces(self.h, _ptr(ts, C.c_uint64), _ptr(cx, C.c_uint32),
                                      _ptr(off, C.c_uint64), _ptr(te, C.c_uint64),
                                      _ptr(pid, C.c_uint32)))
        return {"ts": ts, "ctx": cx, "off": off, "t_end": te, "pid": pid}

    def index(self) -> dict:
        """The trace index only (event offsets, t_end, profile ids)."""
        n = self.shard()["n_traces"]
        off = np.empty(n + 1, np.uint64)
        te = np.empty(n, np.uint64)
        pid = np.empty(n, np.uint32)
        check(self.lib.psg_get_traces(self.h, None, None, _ptr(off, C.c_uint64),
                                      _ptr(te, C.c_uint64), _ptr(pid, C.c_uint32)))
        return {"off": off, "t_end": te, "pid": pid}

    # -- query -----------------------------------------------------------------
    def query(self, flags: int = Q_ALL, t0: int = 0, t1: int = 0, anchor: int = 1, sites=(),
              top_k: int = 0, z_min: float = float("-inf")) -> dict:
        q = _lib.QuerySpec()
        q.flags = flags
        q.t0_ns, q.t1_ns = t0, t1
        q.anchor_ctx = anchor
        self._sites = np.ascontiguousarray(sites, dtype=np.uint32)
        q.site_ctx = _ptr(self._sites, C.c_uint32) if len(self._sites) else None
        q.n_sites = len(self._sites)
        q.top_k = top_k
        q.z_min = z_min
        info = _lib.QueryInfo()
        check(self.lib.psg_query(self.h, C.byref(q), C.byref(info)))
        self.info = {k: getattr(info, k) for k, _ in info._fields_}
        self._flags = flags
        return self.info

    WINDOW_DTYPES = [("count", np.uint64), ("sum", np.int64), ("min", np.int64), ("max", np.int64),
                     ("mean", np.float64), ("excl", np.int64), ("incl", np.int64)]

    def window(self, out: Optional[dict] = None) -> dict:
        """Dense [trace][ctx] window aggregates; `out` may supply the seven host
        arrays (e.g. views of pinned buffers, for a fast copy-out)."""
        sh = self.shard()
        shape = (sh["n_traces"], sh["n_ctx"])
        if out is None:
            out = {k: np.empty(shape, dt) for k, dt in self.WINDOW_DTYPES}
        for k, dt in self.WINDOW_DTYPES:
            a = out[k]
            assert a.dtype == dt and a.size == shape[0] * shape[1] and a.flags.c_contiguous, k
        check(self.lib.psg_get_window(
            self.h, _ptr(out["count"], C.c_uint64), _ptr(out["sum"], C.c_int64),
            _ptr(out["min"], C.c_int64), _ptr(out["max"], C.c_int64),
            _ptr(out["mean"], C.c_double), _ptr(out["excl"], C.c_int64),
            _ptr(out["incl"], C.c_int64)))
        return out

    def window_groups(self) -> dict:
        """group_aggregate rows of the window (count > 0), sorted by (trace, ctx)."""
        n = C.c_uint64(0)
        check(self.lib.psg_get_window_groups(self.h, C.byref(n), None, None, None, None, None, None, None))
        m = n.value
        out = {"trace": np.empty(m, np.uint32), "ctx": np.empty(m, np.uint32), "count": np.empty(m, np.uint64),
               "sum": np.empty(m, np.int64), "min": np.empty(m, np.int64), "max": np.empty(m, np.int64),
               "mean": np.empty(m, np.float64)}
        if m:
            check(self.lib.psg_get_window_groups(
                self.h, C.byref(n), _ptr(out["trace"], C.c_uint32), _ptr(out["ctx"], C.c_uint32),
                _ptr(out["count"], C.c_uint64), _ptr(out["sum"], C.c_int64), _ptr(out["min"], C.c_int64),
                _ptr(out["max"], C.c_int64), _ptr(out["mean"], C.c_double)))
        return out

    def remat_rows(self) -> dict:
        """rematerialize rows of the window (incl or excl nonzero), sorted by (trace, ctx)."""
        n = C.c_uint64(0)
        check(self.lib.psg_get_remat_rows(self.h, C.byref(n), None, None, None, None))
        m = n.value
        out = {"trace": np.empty(m, np.uint32), "ctx": np.empty(m, np.uint32), "incl": np.empty(m, np.int64),
               "excl": np.empty(m, np.int64)}
        if m:
            check(self.lib.psg_get_remat_rows(self.h, C.byref(n), _ptr(out["trace"], C.c_uint32),
                                              _ptr(out["ctx"], C.c_uint32), _ptr(out["incl"], C.c_int64),
                                              _ptr(out["excl"], C.c_int64)))
        return out

    def carry(self) -> dict:
        n = self.shard()["n_traces"]
        has = np.empty(n, np.uint8)
        ts = np.empty(n, np.uint64)
        cx = np.empty(n, np.uint32)
        check(self.lib.psg_get_carry(self.h, _ptr(has, C.c_uint8), _ptr(ts, C.c_uint64),
                                     _ptr(cx, C.c_uint32)))
        return {"has": has, "ts": ts, "ctx": cx}

    def cube(self, with_cells: bool = True, out: Optional[dict] = None) -> dict:
        """The dense cube (reference layout, itermodel.hpp:97-101).  `out` may
        supply host arrays (e.g. views of pinned buffers, for a fast copy-out)
        for "iter_counts", "block_offset", "gap_incl" and "gap_excl" (at least
        n_traces / n_kept / n_kept * n_nodes entries; views of their leading
        parts are returned)."""
        info = self.info
        n = self.shard()["n_traces"]
        nn, kept, cells = info["n_nodes"], info["n_kept"], info["n_cells"]
        out = out or {}

        def arr(key, size, dt):
            a = out.get(key)
            if a is None:
                return np.empty(size, dt)
            assert a.dtype == dt and a.size >= size and a.flags.c_contiguous, key
            return a.reshape(-1)[:size]

        node_ids = np.empty(nn, np.uint32)
        ic = arr("iter_counts", n, np.uint32)
        bo = arr("block_offset", kept, np.uint64)
        incl = np.empty(cells, np.int64) if with_cells else None
        excl = np.empty(cells, np.int64) if with_cells else None
        gi = arr("gap_incl", kept * nn, np.int64)
        ge = arr("gap_excl", kept * nn, np.int64)
        check(self.lib.psg_get_cube(self.h, _ptr(node_ids, C.c_uint32), _ptr(ic, C.c_uint32),
                                    _ptr(bo, C.c_uint64), _ptr(incl, C.c_int64),
                                    _ptr(excl, C.c_int64), _ptr(gi, C.c_int64),
                                    _ptr(ge, C.c_int64)))
        return {"node_ids": node_ids, "iter_counts": ic, "block_offset": bo, "incl": incl,
                "excl": excl, "gap_incl": gi, "gap_excl": ge}

    def cube_range(self, t_lo: int, t_hi: int) -> dict:
        """The dense cube of loaded traces [t_lo, t_hi) (kept ones, in load
        order): incl / excl cells and gap rows, widened on the device."""
        nn = self.info["n_nodes"]
        cells, kept = C.c_uint64(), C.c_uint32()
        check(self.lib.psg_get_cube_range(self.h, t_lo, t_hi, C.byref(cells), C.byref(kept),
                                          None, None, None, None))
        incl = np.empty(cells.value, np.int64)
        excl = np.empty(cells.value, np.int64)
        gi = np.empty(kept.value * nn, np.int64)
        ge = np.empty(kept.value * nn, np.int64)
        check(self.lib.psg_get_cube_range(self.h, t_lo, t_hi, C.byref(cells), C.byref(kept),
                                          _ptr(incl, C.c_int64), _ptr(excl, C.c_int64),
                                          _ptr(gi, C.c_int64), _ptr(ge, C.c_int64)))
        return {"incl": incl, "excl": excl, "gap_incl": gi, "gap_excl": ge, "n_kept": kept.value}

    def cube_stored(self, incl_out: Optional[np.ndarray] = None,
                    xint_out: Optional[np.ndarray] = None, wait: bool = True,
                    off_out: Optional[np.ndarray] = None) -> dict:
        """The cube as stored in HBM, copied without conversion: incl cells
        (uint32 or uint64) in rows of `row_stride`, per-trace stored offsets,
        and the internal nodes' excl.  Pass pinned arrays (e.g. torch
        pin_memory buffers viewed through numpy) to copy at full PCIe rate;
        wait=False returns at once (the arrays fill in the background until
        wait_copies() or the next query)."""
        cb, st, nb, nx = C.c_uint32(), C.c_uint32(), C.c_uint64(), C.c_uint64()
        check(self.lib.psg_get_cube_stored(self.h, C.byref(cb), C.byref(st), C.byref(nb), None, None,
                                           C.byref(nx), None))
        dt = np.uint32 if cb.value == 4 else np.uint64
        incl = incl_out if incl_out is not None else np.empty(nb.value // cb.value, dt)
        assert incl.nbytes >= nb.value, "incl_out too small"
        xint = xint_out if xint_out is not None else np.empty(nx.value, np.int64)
        off = off_out if off_out is not None else np.empty(self.shard()["n_traces"], np.uint64)
        if wait:
            check(self.lib.psg_get_cube_stored(self.h, None, None, None, C.c_void_p(incl.ctypes.data),
                                               _ptr(off, C.c_uint64), None,
                                               _ptr(xint, C.c_int64) if nx.value else None))
        else:
            check(self.lib.psg_get_cube_stored_async(self.h, C.c_void_p(incl.ctypes.data), _ptr(off, C.c_uint64),
                                                     _ptr(xint, C.c_int64) if nx.value else None))
        return {"incl": incl.view(dt)[: nb.value // cb.value], "xint": xint[: nx.value],
                "stored_off": off, "row_stride": st.value, "cell_bytes": cb.value}

    def wait_copies(self):
        """Block until an asynchronous copy-out (cube_stored(wait=False)) landed."""
        check(self.lib.psg_wait_copies(self.h))

    def stats(self, total_time_s: float) -> dict:
        nl = self.info["n_leaves"]
        leaves = np.empty(nl, np.uint32)
        sav = np.empty((nl, 4), np.float64)
        summ = np.empty(4, np.float64)
        cv = np.empty((nl, 2), np.float64)
        ok = np.empty(nl, np.int32)
        check(self.lib.psg_get_stats(self.h, total_time_s, _ptr(leaves, C.c_uint32),
                                     _ptr(sav, C.c_double), _ptr(summ, C.c_double),
                                     _ptr(cv, C.c_double), _ptr(ok, C.c_int32)))
        return {"leaves": leaves, "savings": sav, "summary": summ, "cv": cv, "cv_ok": ok}

    def outliers(self, n_nodes: int, masks: bool = True) -> dict:
        info = self.info
        ns = len(self._sites)
        ratio = np.empty(ns, np.float64)
        mean = np.empty(n_nodes, np.float64)
        z = np.empty(n_nodes, np.float64)
        sel = np.empty(max(1, info["n_outliers"]), np.uint32)
        nr = info["n_racks"]
        rows = np.empty((max(1, nr), 3), np.uint32)
        cm = np.empty(max(1, nr), np.uint64)
        fm = np.empty(max(1, nr), np.uint64)
        check(self.lib.psg_get_outliers(self.h, _ptr(ratio, C.c_double), _ptr(mean, C.c_double),
                                        _ptr(z, C.c_double), _ptr(sel, C.c_uint32),
                                        _ptr(rows, C.c_uint32),
                                        _ptr(cm, C.c_uint64) if masks else None,
                                        _ptr(fm, C.c_uint64) if masks else None))
        out = {"site_ratio": ratio, "node_mean": mean, "node_z": z,
               "selected": sel[: info["n_outliers"]], "racks": rows[:nr]}
        if masks:
            out["chassis_mask"], out["full_mask"] = cm[:nr], fm[:nr]
        return out

    def topology(self) -> np.ndarray:
        """localize_outliers rows [rack, chassis, outlier nodes, fully affected]."""
        n = C.c_uint32(0)
        check(self.lib.psg_get_topology(self.h, C.byref(n), None))
        rows = np.empty((max(1, n.value), 4), np.uint32)
        check(self.lib.psg_get_topology(self.h, C.byref(n), _ptr(rows, C.c_uint32)))
        return rows[: n.value]

    # ---- profile records (profile.db) -----------------------------------
    def load_profiles(self, records, rec_off, pids, ranks, node_of_profile=None):
        """records: uint8 array of packed 14-byte {u32 ctx, u16 metric, f64} records."""
        off = np.ascontiguousarray(rec_off, dtype=np.uint64)
        pid = np.ascontiguousarray(pids, dtype=np.uint32)
        rk = np.ascontiguousarray(ranks, dtype=np.int32)
        rec = np.ascontiguousarray(records, dtype=np.uint8)
        nd = None if node_of_profile is None else np.ascontiguousarray(node_of_profile, dtype=np.uint32)
        check(self.lib.psg_load_profiles(self.h, C.c_void_p(rec.ctypes.data if rec.size else 0),
                                         _ptr(off, C.c_uint64), _ptr(pid, C.c_uint32), _ptr(rk, C.c_int32),
                                         _ptr(nd, C.c_uint32) if nd is not None else None, len(pid)))

    def load_profile_db(self, path: str):
        check(self.lib.psg_load_profile_db(self.h, path.encode()))

    def slice(self, pids, ctx_ids=None, metric_ids=None) -> dict:
        """ingest_profiles / read_slices: rows (pid, ctx, metric, value)."""
        p = np.ascontiguousarray(pids, dtype=np.uint32)
        cx = None if ctx_ids is None else np.ascontiguousarray(ctx_ids, dtype=np.uint32)
        mt = None if metric_ids is None else np.ascontiguousarray(metric_ids, dtype=np.uint16)
        args = [self.h, _ptr(p, C.c_uint32), len(p),
                _ptr(cx, C.c_uint32) if cx is not None else None, 0 if cx is None else len(cx),
                _ptr(mt, C.c_uint16) if mt is not None else None, 0 if mt is None else len(mt)]
        n = C.c_uint64()
        check(self.lib.psg_slice(*args, C.byref(n), None, None, None, None))
        m = n.value
        out = {"pid": np.empty(max(1, m), np.uint32), "ctx": np.empty(max(1, m), np.uint32),
               "metric": np.empty(max(1, m), np.uint16), "value": np.empty(max(1, m), np.float64)}
        check(self.lib.psg_slice(*args, C.byref(n), _ptr(out["pid"], C.c_uint32),
                                 _ptr(out["ctx"], C.c_uint32), _ptr(out["metric"], C.c_uint16),
                                 _ptr(out["value"], C.c_double)))
        return {k: v[:m] for k, v in out.items()}

    def profile_outliers(self, metric: int, sites, top_k: int = 0, z_min: float = float("-inf")) -> dict:
        self._sites = np.ascontiguousarray(sites, dtype=np.uint32)
        info = _lib.QueryInfo()
        check(self.lib.psg_profile_outliers(self.h, metric, _ptr(self._sites, C.c_uint32),
                                            len(self._sites), top_k, z_min, C.byref(info)))
        self.info = {k: getattr(info, k) for k, _ in info._fields_}
        return self.info

    def export_aos(self, body_addr: int):
        """Writes the loaded traces as packed trace.db bytes to host address body_addr."""
        check(self.lib.psg_export_aos(self.h, C.c_void_p(body_addr)))

    def export_aos_range(self, t_lo: int, t_hi: int) -> np.ndarray:
        """Traces [t_lo, t_hi) as packed trace.db bytes (uint8 array)."""
        idx = self.index()
        n = int(idx["off"][t_hi] - idx["off"][t_lo])
        body = np.empty(max(1, n * 12), np.uint8)
        check(self.lib.psg_export_aos_range(self.h, t_lo, t_hi, C.c_void_p(body.ctypes.data)))
        return body[: n * 12]

    @staticmethod
    def kernel_launches() -> int:
        return int(load().psg_kernel_launches())

    def window_row_count(self, t0: int, t1: int) -> int:
        """Rows of ingest_traces' window (psg_window_rows' size query only)."""
        n = C.c_uint64()
        check(self.lib.psg_window_rows(self.h, t0, t1, C.byref(n), None, None, None))
        return n.value

    def window_rows(self, t0: int, t1: int) -> dict:
        n = C.c_uint64()
        check(self.lib.psg_window_rows(self.h, t0, t1, C.byref(n), None, None, None))
        m = n.value
        pid = np.empty(max(1, m), np.uint32)
        ts = np.empty(max(1, m), np.uint64)
        cx = np.empty(max(1, m), np.uint32)
        check(self.lib.psg_window_rows(self.h, t0, t1, C.byref(n), _ptr(pid, C.c_uint32),
                                       _ptr(ts, C.c_uint64), _ptr(cx, C.c_uint32)))
        out = {"pid": pid[:m], "ts": ts[:m], "ctx": cx[:m]}
        out["carry"] = self.carry()
        return out

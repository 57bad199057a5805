"""GPU frame operators: the reference's columnar engine (frame.hpp) for numeric
columns on the device, with its determinism contract (every result equals the
reference's bit for bit).  Columns are CUDA tensors (i64 / u64 / f64; u64 is
held in an int64 tensor with the same bits); the work runs in libpsg.so
(csrc/psg_frame.cu) on the context's stream.

    t = frame.Table(ctx); t.add("pid", pid_tensor, "u64"); ...
    frame.group_aggregate(t, ["pid", "ctx"], [("dur", "sum"), ("dur", "max")])
    frame.sort(t, ["ts"]), frame.filter(t, "ts", "ge", 5), frame.merge(a, b, ["pid"])
    frame.reduce_sum(ctx, col), frame.cumulative_sum(ctx, col), ...
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _lib
from ._lib import check

DTYPES = {"i64": 0, "u64": 1, "f64": 2}
OPS = {"lt": 0, "le": 1, "eq": 2, "ge": 3, "gt": 4, "ne": 5}
AGGS = {"sum": 0, "min": 1, "max": 2, "mean": 3, "count": 4}
AGG_DTYPE = {"mean": "f64", "count": "u64"}


class Column:
    def __init__(self, name: str, data: torch.Tensor, dtype: str):
        if dtype not in DTYPES:
            raise ValueError("dtype must be i64, u64 or f64 (strings stay on the host)")
        want = torch.float64 if dtype == "f64" else torch.int64
        if not data.is_cuda or data.dtype != want or data.dim() != 1:
            raise ValueError(f"column {name}: a 1-D CUDA {want} tensor is required")
        self.name, self.data, self.dtype = name, data.contiguous(), dtype

    def __len__(self) -> int:
        return self.data.numel()

    def c(self) -> _lib.PsgCol:
        return _lib.PsgCol(DTYPES[self.dtype], self.data.data_ptr())

    def numpy(self) -> np.ndarray:
        a = self.data.cpu().numpy()
        return a.view(np.uint64) if self.dtype == "u64" else a

    @staticmethod
    def from_numpy(name: str, a: np.ndarray, device: str = "cuda") -> "Column":
        dt = {np.dtype(np.int64): "i64", np.dtype(np.uint64): "u64", np.dtype(np.float64): "f64"}[a.dtype]
        t = torch.from_numpy(np.ascontiguousarray(a).view(np.float64 if dt == "f64" else np.int64).copy())
        return Column(name, t.to(device), dt)


class Table:
    def __init__(self, ctx):
        self.ctx = ctx
        self.cols: Dict[str, Column] = {}

    def add(self, name: str, data: torch.Tensor, dtype: str) -> "Table":
        if name in self.cols:
            raise ValueError(f"duplicate column {name}")
        if self.cols and len(data) != self.n_rows():
            raise ValueError("column length mismatch")
        self.cols[name] = Column(name, data, dtype)
        return self

    def add_column(self, c: Column) -> "Table":
        return self.add(c.name, c.data, c.dtype)

    def n_rows(self) -> int:
        return len(next(iter(self.cols.values()))) if self.cols else 0

    def col(self, name: str) -> Column:
        if name not in self.cols:
            raise KeyError(f"no such column: {name}")
        return self.cols[name]

    def gather(self, idx: torch.Tensor) -> "Table":
        out = Table(self.ctx)
        for c in self.cols.values():
            out.add_column(_gather(self.ctx, c, idx))
        return out


def _h(ctx):
    return ctx.h


def _lib_of(ctx):
    return ctx.lib


def _cols(cols: Sequence[Column]):
    arr = (_lib.PsgCol * max(1, len(cols)))(*[c.c() for c in cols])
    return arr


def _gather(ctx, c: Column, idx: torch.Tensor) -> Column:
    out = torch.empty(idx.numel(), dtype=c.data.dtype, device=c.data.device)
    check(ctx.lib.psg_frame_gather(ctx.h, c.c(), C.c_void_p(idx.data_ptr()), idx.numel(),
                                   C.c_void_p(out.data_ptr())))
    return Column(c.name, out, c.dtype)


def argsort(ctx, keys: Sequence[Column], ascending: Optional[Sequence[bool]] = None) -> torch.Tensor:
    n = len(keys[0]) if keys else 0
    perm = torch.empty(max(1, n), dtype=torch.int64, device="cuda")
    asc = None
    if ascending is not None:
        if len(ascending) != len(keys):
            raise ValueError("ascending flags do not match key count")
        asc = np.array([1 if a else 0 for a in ascending], np.uint8)
    check(ctx.lib.psg_frame_argsort(ctx.h, _cols(keys), len(keys),
                                    asc.ctypes.data_as(C.POINTER(C.c_uint8)) if asc is not None else None,
                                    n, C.c_void_p(perm.data_ptr())))
    return perm[:n]


def sort(t: Table, keys: Sequence[str], ascending: Optional[Sequence[bool]] = None) -> Table:
    """frame::sort (frame.cpp:410-422): stable multi-key sort of every column."""
    perm = argsort(t.ctx, [t.col(k) for k in keys], ascending)
    return t.gather(perm)


def group_aggregate(t: Table, keys: Sequence[str], aggs: Sequence[Tuple[str, str]]) -> Table:
    """frame::group_aggregate (frame.cpp:290-408): one row per distinct key
    tuple, ascending; aggregate columns named <column>_<fn>."""
    ctx, n = t.ctx, t.n_rows()
    kc = [t.col(k) for k in keys]
    perm = torch.empty(max(1, n), dtype=torch.int64, device="cuda")
    starts = torch.empty(max(1, n), dtype=torch.int64, device="cuda")
    ng = C.c_uint64()
    check(ctx.lib.psg_frame_group(ctx.h, _cols(kc), len(kc), n, C.c_void_p(perm.data_ptr()),
                                  C.c_void_p(starts.data_ptr()), C.byref(ng)))
    g = ng.value
    heads = perm[starts[:g]] if g else perm[:0]
    out = Table(ctx)
    for c in kc:
        out.add_column(_gather(ctx, c, heads))
    for name, fn in aggs:
        src = t.col(name)
        dt = AGG_DTYPE.get(fn, src.dtype)
        res = torch.empty(max(1, g), dtype=torch.float64 if dt == "f64" else torch.int64, device="cuda")
        check(ctx.lib.psg_frame_group_agg(ctx.h, src.c(), C.c_void_p(perm.data_ptr()),
                                          C.c_void_p(starts.data_ptr()), g, n, AGGS[fn],
                                          C.c_void_p(res.data_ptr())))
        out.add(f"{name}_{fn}", res[:g], dt)
    return out


def filter(t: Table, column: str, op: str, literal) -> Table:  # noqa: A001 (the reference's name)
    """frame::filter (frame.cpp:424-470): rows with (column <op> literal), in order."""
    ctx, n, c = t.ctx, t.n_rows(), t.col(column)
    lit = np.array([literal], {"i64": np.int64, "u64": np.uint64, "f64": np.float64}[c.dtype])
    idx = torch.empty(max(1, n), dtype=torch.int64, device="cuda")
    m = C.c_uint64()
    check(ctx.lib.psg_frame_filter(ctx.h, c.c(), OPS[op], C.c_void_p(lit.ctypes.data), n,
                                   C.c_void_p(idx.data_ptr()), C.byref(m)))
    return t.gather(idx[:m.value])


def merge(left: Table, right: Table, on: Sequence[str]) -> Table:
    """frame::merge (frame.cpp:472-572): inner join ordered by (left row, right
    row); right non-key columns appended, "_r" suffixed on a name collision."""
    ctx = left.ctx
    lk, rk = [left.col(k) for k in on], [right.col(k) for k in on]
    n = C.c_uint64()
    check(ctx.lib.psg_frame_merge(ctx.h, _cols(lk), _cols(rk), len(on), left.n_rows(), right.n_rows(), 0,
                                  None, None, C.byref(n)))
    m = n.value
    li = torch.empty(max(1, m), dtype=torch.int64, device="cuda")
    ri = torch.empty(max(1, m), dtype=torch.int64, device="cuda")
    check(ctx.lib.psg_frame_merge(ctx.h, _cols(lk), _cols(rk), len(on), left.n_rows(), right.n_rows(), m,
                                  C.c_void_p(li.data_ptr()), C.c_void_p(ri.data_ptr()), C.byref(n)))
    out = Table(ctx)
    for c in left.cols.values():
        out.add_column(_gather(ctx, c, li[:m]))
    for c in right.cols.values():
        if c.name in on:
            continue
        g = _gather(ctx, c, ri[:m])
        if g.name in out.cols:
            g.name += "_r"
        out.add_column(g)
    return out


def _f64(c: Column):
    if c.dtype != "f64":
        raise TypeError(f"column {c.name} must be f64")
    return C.c_void_p(c.data.data_ptr())


def vector_add(ctx, a: Column, b: Column) -> Column:
    if len(a) != len(b):
        raise ValueError("vector_add length mismatch")
    out = torch.empty_like(a.data)
    check(ctx.lib.psg_frame_vector_add(ctx.h, _f64(a), _f64(b), len(a), C.c_void_p(out.data_ptr())))
    return Column(a.name, out, "f64")


def in_place_multiply(ctx, a: Column, scalar: float) -> Column:
    out = torch.empty_like(a.data)
    check(ctx.lib.psg_frame_multiply(ctx.h, _f64(a), scalar, len(a), C.c_void_p(out.data_ptr())))
    return Column(a.name, out, "f64")


def scalar_compare(ctx, a: Column, op: str, scalar: float) -> Column:
    out = torch.empty(len(a), dtype=torch.int64, device="cuda")
    check(ctx.lib.psg_frame_scalar_compare(ctx.h, _f64(a), OPS[op], scalar, len(a), C.c_void_p(out.data_ptr())))
    return Column(a.name, out, "i64")


def reduce_sum(ctx, a: Column) -> float:
    r = C.c_double()
    check(ctx.lib.psg_frame_reduce_sum(ctx.h, _f64(a), len(a), C.byref(r)))
    return r.value


def cumulative_sum(ctx, a: Column) -> Column:
    out = torch.empty_like(a.data)
    check(ctx.lib.psg_frame_cumsum(ctx.h, _f64(a), len(a), C.c_void_p(out.data_ptr())))
    return Column(a.name, out, "f64")

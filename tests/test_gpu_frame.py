"""GPU frame operators (the paper's Query API op set,
PAPER.md Tables 1-3) against the reference's frame engine (oracle/_ref), bit
for bit: sort, group_aggregate, filter, merge, vector_add, in_place_multiply,
scalar_compare, reduce_sum, cumulative_sum."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from paper_2605_03561_b200 import PsgError, frame

pytestmark = pytest.mark.gpu


def inputs(seed: int, n: int):
    rng = np.random.default_rng(seed)
    a = rng.integers(-6, 6, n).astype(np.int64)
    b = rng.random(n)
    b[::7] = np.nan
    b[::11] = -0.0
    b[::13] = 0.0
    c = rng.integers(0, 4, n).astype(np.uint64)
    v = rng.random(n) * 100 - 50
    w = rng.integers(-(2**62), 2**62, n).astype(np.int64)
    return a, b, c, v, w


def table(ctx, **cols) -> frame.Table:
    t = frame.Table(ctx)
    for name, arr in cols.items():
        t.add_column(frame.Column.from_numpy(name, arr))
    return t


@pytest.mark.parametrize("n", [0, 1, 1000, 70_000])
def test_sort_and_filter(gpu_ctx_factory, n):
    ctx = gpu_ctx_factory()
    a, b, c, v, w = inputs(n, n)
    t = table(ctx, a=a, b=b, c=c, row=np.arange(n, dtype=np.uint64))
    for keys, asc in ((["a"], None), (["b", "c"], None), (["a", "b", "c"], [True, False, True]),
                      (["c", "b"], [False, False])):
        want = oracle.ref_frame_sort([{"a": a, "b": b, "c": c}[k] for k in keys], asc)
        s = frame.sort(t, keys, asc)
        assert np.array_equal(s.col("row").numpy(), want), (keys, asc)
    for col, op, lit in (("b", "ge", 0.5), ("b", "ne", 0.25), ("b", "eq", 0.0), ("a", "lt", 0),
                         ("c", "eq", 2), ("b", "gt", float("nan"))):
        arr = {"a": a, "b": b, "c": c}[col]
        want = oracle.ref_frame_filter(arr, op, lit)
        f = frame.filter(t, col, op, lit)
        assert np.array_equal(f.col("row").numpy(), want), (col, op, lit)


@pytest.mark.parametrize("n", [2_000_003])
def test_sort_large_multi_tile(gpu_ctx_factory, n):
    """The hand-written radix sort (psg_sort.cu) across many tiles and all
    eight digit passes: full-range int64 keys, few-valued keys with long runs
    of ties (stability), descending order, and NaN / -0.0 doubles."""
    ctx = gpu_ctx_factory()
    a, b, c, v, w = inputs(7, n)
    t = table(ctx, a=a, b=b, c=c, w=w, row=np.arange(n, dtype=np.uint64))
    for keys, asc in ((["w"], None), (["c"], [False]), (["a", "w"], [True, False]), (["b", "c"], None)):
        want = oracle.ref_frame_sort([{"a": a, "b": b, "c": c, "w": w}[k] for k in keys], asc)
        s = frame.sort(t, keys, asc)
        assert np.array_equal(s.col("row").numpy(), want), (keys, asc)


@pytest.mark.parametrize("n", [1, 5000, 100_000])
def test_group_aggregate(gpu_ctx_factory, n):
    ctx = gpu_ctx_factory()
    a, b, c, v, w = inputs(100 + n, n)
    t = table(ctx, a=a, b=b, c=c, v=v, w=w, u=c * np.uint64(3))
    for keys in (["a"], ["c", "a"], ["b"], ["a", "b", "c"]):
        for src, fn in (("v", "sum"), ("v", "mean"), ("v", "min"), ("v", "max"), ("w", "sum"),
                        ("w", "max"), ("u", "min"), ("u", "sum"), ("a", "mean"), ("v", "count")):
            g = frame.group_aggregate(t, keys, [(src, fn)])
            src_arr = {"v": v, "w": w, "u": c * np.uint64(3), "a": a}[src]
            wk, wa = oracle.ref_frame_group([{"a": a, "b": b, "c": c}[k] for k in keys], src_arr, fn)
            for k, want in zip(keys, wk):
                got = g.col(k).numpy()
                assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (keys, src, fn, k)
            got = g.col(f"{src}_{fn}").numpy()
            assert np.array_equal(got.view(np.uint64), wa.view(np.uint64)), (keys, src, fn)
    # require_numeric: NaN in an aggregate column raises (frame.cpp:150-156)
    with pytest.raises(PsgError):
        frame.group_aggregate(table(ctx, k=np.zeros(3, np.int64), x=np.array([1.0, np.nan, 2.0])), ["k"],
                              [("x", "sum")])


@pytest.mark.parametrize("seed", range(3))
def test_merge(gpu_ctx_factory, seed):
    ctx = gpu_ctx_factory()
    rng = np.random.default_rng(seed)
    nl, nr = 3000, 2000
    la, ra = rng.integers(0, 300, nl).astype(np.int64), rng.integers(0, 300, nr).astype(np.int64)
    lb, rb = rng.random(nl).round(1), rng.random(nr).round(1)
    lt = table(ctx, k=la, f=lb, lrow=np.arange(nl, dtype=np.uint64), x=rng.random(nl))
    rt = table(ctx, k=ra, f=rb, rrow=np.arange(nr, dtype=np.uint64), x=rng.random(nr))
    for on in (["k"], ["k", "f"]):
        m = frame.merge(lt, rt, on)
        wl, wr = oracle.ref_frame_merge([{"k": la, "f": lb}[k] for k in on], [{"k": ra, "f": rb}[k] for k in on])
        assert np.array_equal(m.col("lrow").numpy(), wl) and np.array_equal(m.col("rrow").numpy(), wr), on
        assert "x_r" in m.cols and ("f_r" in m.cols) == ("f" not in on)


@pytest.mark.parametrize("n", [1, 4096, 4097, 1_000_003])
def test_vector_ops_bit_exact(gpu_ctx_factory, n):
    ctx = gpu_ctx_factory()
    rng = np.random.default_rng(n)
    x, y = rng.random(n) * 1e6 - 3e5, rng.random(n) * 7 - 1
    x[::97] = np.nan
    X, Y = frame.Column.from_numpy("x", x), frame.Column.from_numpy("y", y)
    same = lambda g, r: np.array_equal(np.asarray(g).view(np.uint64), np.asarray(r).view(np.uint64))  # noqa: E731
    assert same(frame.vector_add(ctx, X, Y).numpy(), oracle.ref_frame_vec("vector_add", x, y))
    assert same(frame.in_place_multiply(ctx, X, 1.7).numpy(), oracle.ref_frame_vec("multiply", x, scalar=1.7))
    for op in ("lt", "le", "eq", "ge", "gt", "ne"):
        assert np.array_equal(frame.scalar_compare(ctx, X, op, 0.25).numpy(),
                              oracle.ref_frame_vec("scalar_compare", x, scalar=0.25, cmp=op)), op
    z = np.where(np.isnan(x), 1.0, x)
    Z = frame.Column.from_numpy("z", z)
    assert same([frame.reduce_sum(ctx, Z)], [oracle.ref_frame_vec("reduce_sum", z)])
    cs = frame.cumulative_sum(ctx, Z).numpy()
    assert same(cs, oracle.ref_frame_vec("cumsum", z))
    assert cs[-1] == frame.reduce_sum(ctx, Z)

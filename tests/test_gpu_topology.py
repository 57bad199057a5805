"""GPU: the topology half of the outlier path (K8) against the reference's
topology::localize_outliers (topology.cpp:14-92), including what round 1
missed: chassis ids >= 64 (any id, as long as a rack has <= 64 distinct
chassis) and the parse_error the reference raises for a hostname that is not
a Slingshot x<r>c<c>s<s>b<b>n<n> name (appendix trap 12)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from paper_2605_03561_b200 import Q_CLAMP_TEND, Q_OUTLIERS, Q_WINDOW, PsgError, scenarios
from paper_2605_03561_b200._lib import STATUS_NAMES
from tests.helpers import ref_db

pytestmark = pytest.mark.gpu
PS_E_PARSE = STATUS_NAMES.index("parse_error")
PS_E_INVALID_ARGUMENT = STATUS_NAMES.index("invalid_argument")


def _hosts(rack, chassis):
    return [f"x{r}c{c}s{i % 8}b0n{i}" for i, (r, c) in enumerate(zip(rack, chassis))]


def test_topology_rows_equal_localize_outliers_any_chassis_id(gpu_ctx_factory):
    ctx = gpu_ctx_factory()
    n_tr, n_nodes = 96, 24
    ctx.generate_iterative(scenarios.iterative(n_tr, 6, n_kernels=4, seed=9, jitter=0.3))
    T = int(ctx.shard()["t_max"])
    rng = np.random.default_rng(4)
    node_of = np.arange(n_tr) // (n_tr // n_nodes)
    rack = 3000 + (np.arange(n_nodes) % 5)
    chassis = rng.choice([0, 7, 63, 64, 100, 4095, 70000], size=n_nodes)
    ctx.set_nodes(node_of, n_nodes, rack, chassis)
    ctx.query(Q_WINDOW | Q_OUTLIERS, t0=0, t1=T, sites=[2, 3], top_k=11)
    out = ctx.outliers(n_nodes, masks=False)
    # localize_outliers is order-free (a set of outliers, maps by rack and
    # chassis), so the universe may be listed in node-id order
    hosts = _hosts(rack, chassis)
    want = oracle.ref_localize([hosts[i] for i in out["selected"]], hosts)
    rows = ctx.topology()
    got = {}
    for r, c, k, full in rows.tolist():
        got.setdefault(r, {"nodes": 0, "chassis": [], "full": []})
        got[r]["nodes"] += k
        got[r]["chassis"].append(c)
        if full:
            got[r]["full"].append(c)
    assert [e["rack"] for e in want["racks"]] == sorted(got)
    for e in want["racks"]:
        g = got[e["rack"]]
        assert g["nodes"] == e["nodes"] and g["chassis"] == e["chassis"] and g["full"] == e["full_chassis"]
    assert [int(r[0]) for r in out["racks"]] == [e["rack"] for e in want["racks"]]
    assert [int(r[1]) for r in out["racks"]] == [e["nodes"] for e in want["racks"]]
    # the u64 masks cannot name chassis >= 64
    if any(c >= 64 for e in want["racks"] for c in e["chassis"]):
        with pytest.raises(PsgError) as ei:
            ctx.outliers(n_nodes, masks=True)
        assert ei.value.status == PS_E_INVALID_ARGUMENT


def test_topology_masks_are_chassis_ids_below_64(gpu_ctx_factory):
    ctx = gpu_ctx_factory()
    n_tr, n_nodes = 64, 16
    ctx.generate_iterative(scenarios.iterative(n_tr, 5, n_kernels=4, seed=2, jitter=0.3))
    T = int(ctx.shard()["t_max"])
    node_of = np.arange(n_tr) // 4
    rack = 4000 + np.arange(n_nodes) // 8
    chassis = np.array([0, 2, 5, 63] * 4)
    ctx.set_nodes(node_of, n_nodes, rack, chassis)
    ctx.query(Q_WINDOW | Q_OUTLIERS, t0=0, t1=T, sites=[2], top_k=6)
    out = ctx.outliers(n_nodes)
    hosts = _hosts(rack, chassis)
    want = oracle.ref_localize([hosts[i] for i in out["selected"]], hosts)
    for j, e in enumerate(want["racks"]):
        assert int(out["chassis_mask"][j]) == sum(1 << c for c in e["chassis"])
        assert int(out["full_mask"][j]) == sum(1 << c for c in e["full_chassis"])


@pytest.mark.parametrize("bad", ["nid001234", "x1000c0s0b0", "x1000cAs0b0n0", "x1000c0s0b0n0-eth"])
def test_trace_db_bad_hostname_raises_parse_error(gpu_ctx_factory, bad):
    """psg_load_trace_db / psg_load_profile_db over a database the reference
    wrote with a non-Slingshot hostname: loading and window queries work; an
    outlier query raises PS_E_PARSE with the message localize_outliers raises
    for the same universe (topology.cpp:14-46, appendix trap 12)."""
    cfg = dict(scenarios.iterative(8, 4, n_kernels=3, seed=1), hostname=bad)
    d = ref_db(cfg)
    with pytest.raises(RuntimeError) as ref_err:
        oracle.ref_localize([], [bad])
    want = str(ref_err.value).split(": ", 1)[1]
    ctx = gpu_ctx_factory()
    ctx.load_trace_db(d)
    T = int(ctx.shard()["t_max"])
    ctx.query(Q_WINDOW, t0=0, t1=T)
    with pytest.raises(PsgError) as ei:
        ctx.query(Q_WINDOW | Q_OUTLIERS | Q_CLAMP_TEND, t0=0, t1=T, sites=[2], top_k=1)
    assert ei.value.status == PS_E_PARSE
    assert str(ei.value) == "parse_error: " + want
    ctx.load_profile_db(d)
    with pytest.raises(PsgError) as ei2:
        ctx.profile_outliers(0, [2], 1, 0.0)
    assert ei2.value.status == PS_E_PARSE and str(ei2.value) == "parse_error: " + want

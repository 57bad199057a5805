"""GPU parity of the profile-record path: profile.db
bodies in HBM, the Query API slice (ingest_profiles / read_slices) and
congestion_report's numeric core over profile records, against the reference
(oracle/_ref) and the golden fixture."""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

import oracle
from paper_2605_03561_b200 import PsgError, scenarios
from tests.helpers import GOLDEN, assert_rel

pytestmark = pytest.mark.gpu


def load(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def test_slices_match_ingest_profiles_fixture(gpu_ctx_factory):
    g = load("profiles_rpn1")
    ctx = gpu_ctx_factory()
    rank = g["prof_rank"][np.searchsorted(g["prof_pid"], g["pid"])]
    ctx.load_profiles(g["body"], g["rec_off"], g["pid"], rank)
    for pre, cx, mt in (("all_", None, None), ("filt_", g["req_ctx"], [1])):
        s = ctx.slice(g["req_pids"], cx, mt)
        for k in ("pid", "ctx", "metric", "value"):
            assert np.array_equal(s[k], g[pre + k]), f"{pre}{k}"
    # duplicate and unsorted requests are deduplicated and sorted (ingest.cpp:161-163)
    s = ctx.slice(np.concatenate([g["req_pids"][::-1], g["req_pids"][:3]]), cx, mt)
    assert np.array_equal(s["pid"], g["filt_pid"]) and np.array_equal(s["value"], g["filt_value"])
    with pytest.raises(PsgError) as e:
        ctx.slice([int(g["pid"].max()) + 1])
    assert e.value.name == "not_found"


def test_slices_match_reference_db(gpu_ctx_factory, tmp_path):
    cfg = scenarios.aurora(ranks_per_node=2, seed=7)
    d = str(tmp_path / "db")
    truth = oracle.ref_generate(cfg, d)
    ctx = gpu_ctx_factory()
    ctx.load_profile_db(d)
    meta = oracle.read_meta(d)
    pids = [p for (p, _, _) in meta["profiles"]]
    rng = np.random.default_rng(3)
    for req, cx, mt in ((pids, None, None),
                        (list(rng.choice(pids, 300, replace=False)), sorted(truth["callsite_ctx"]), [1]),
                        (pids[:40], [0], None), (pids[5:9], [], [0, 1])):
        r = oracle.ref_slices(d, req, cx, mt)
        s = ctx.slice(req, cx, mt)
        for k in ("pid", "ctx", "metric", "value"):
            assert np.array_equal(s[k], r[k]), k


def test_profile_congestion_matches_reference(gpu_ctx_factory, tmp_path):
    """C4 shape (aurora_like_config) from profile.db, as congestion_report reads
    it: call-site balance ratios, the worst site, and the z >= 1 / top-202 node
    selection equal the reference's DBSCAN outlier group; racks = the 22."""
    cfg = scenarios.aurora(ranks_per_node=10, seed=2025)
    d = str(tmp_path / "db")
    truth = oracle.ref_generate(cfg, d)
    rep = json.loads(oracle.ref_congestion_report(d))
    meta = oracle.read_meta(d)
    metric = next(m for (m, scope, name) in meta["metrics"] if name == "cputime" and scope == 1)
    ctx = gpu_ctx_factory()
    ctx.load_profile_db(d)
    sites = truth["callsite_ctx"]
    info = ctx.profile_outliers(metric, sites, top_k=0, z_min=1.0)
    assert info["worst_site"] == rep["worst"]["ctx_id"] == truth["congested_ctx"]
    assert abs(info["worst_ratio"] - rep["worst"]["balance_ratio"]) <= 1e-9 * rep["worst"]["balance_ratio"]
    hosts = sorted({h for (_, r, h) in meta["profiles"] if r >= 0})
    out = ctx.outliers(len(hosts))
    assert_rel(out["site_ratio"], [s["balance_ratio"] for s in rep["callsites"]], 1e-9, "balance ratios")
    pdb = oracle.read_profile_db(d)
    o = oracle.profile_sites(pdb, meta, metric, sites)
    assert o["hosts"] == hosts
    assert_rel(out["node_mean"], o["node_mean"], 1e-12, "node means")
    got = sorted(hosts[i] for i in out["selected"])
    assert got == sorted(rep["outlier_group"]["hostnames"]) == sorted(truth["outlier_hostnames"])
    racks = [int(r[0]) for r in out["racks"]]
    assert racks == [r["rack"] for r in rep["topology"]["racks"]] == truth["outlier_rack_ids"]
    info = ctx.profile_outliers(metric, sites, top_k=len(got))
    out2 = ctx.outliers(len(hosts))
    assert sorted(hosts[i] for i in out2["selected"]) == got


def test_profile_records_must_be_ctx_sorted(gpu_ctx_factory):
    rec = np.dtype([("ctx", "<u4"), ("metric", "<u2"), ("value", "<f8")])
    r = np.array([(3, 0, 1.0), (1, 0, 2.0)], dtype=rec)
    ctx = gpu_ctx_factory()
    with pytest.raises(PsgError) as e:
        ctx.load_profiles(np.frombuffer(r.tobytes(), np.uint8), [0, 2], [7], [0])
    assert e.value.name == "format_error"

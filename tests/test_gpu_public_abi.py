"""GPU: the reference's public C ABI with the GPU underneath (SURVEY.md §8(b)
"keep verbatim").  integration/build_public_abi.sh compiles the reference's
own sources into libperfslice.so with the two hot call sites INTEGRATION.md
switches (session cache misses -> gpu::read_slices on psg_slice;
build_tri_model -> gpu::build_tri_model on psg_query, automatic anchor
included).  ps_iterations (capi.cpp:220-232), ps_congestion (:234-250) and
ps_imbalance (:207-218) must return byte-identical CSV / JSON text, and the
same status and message on errors, as the stock reference library."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

from paper_2605_03561_b200 import scenarios
from tests.helpers import ROOT, ref_db

pytestmark = pytest.mark.gpu

STOCK = os.path.join(ROOT, "oracle", "_ref", "libperfslice.so")
GPU = os.path.join(ROOT, "integration", "_build", "public_abi", "libperfslice.so")
CSV, JSON = 0, 1


def _run(lib, db, calls):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "public_abi_worker.py"), lib, db,
                        json.dumps(calls)], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def _same(db, calls):
    ra, rb = _run(STOCK, db, calls), _run(GPU, db, calls)
    # the GPU build really ran the device path; the stock one has no libpsg
    assert ra["psg_kernel_launches"] is None and rb["psg_kernel_launches"] > 0
    a, b = ra["results"], rb["results"]
    assert len(a) == len(b) == len(calls)
    for x, y in zip(a, b):
        assert x["status"] == y["status"], (x["call"], x["text"][:300], y["text"][:300])
        assert x["text"] == y["text"], x["call"]
    return a


@pytest.mark.parametrize("cfg", ["small", "iter_gamess", "iter_ladder"])
def test_ps_iterations_and_imbalance_byte_identical(cfg):
    c = {"small": scenarios.small(seed=31, n_ranks=6, n_iterations=8, jitter=0.2),
         "iter_gamess": scenarios.iterative(48, 20, n_kernels=12, spread="gamess", seed=4),
         "iter_ladder": scenarios.iterative(64, 15, n_kernels=16, seed=6, jitter=0.3)}[cfg]
    db = ref_db(c)
    calls = []
    for fmt in (CSV, JSON):
        for anchor in ("auto", "1", "root", "999999"):
            calls.append(["iterations", anchor, 0.0, fmt])
        calls.append(["iterations", "1", 123.5, fmt])
        calls.append(["imbalance", "gker", 0.01, fmt])
        calls.append(["imbalance", "gker", 0.2, fmt])
        calls.append(["imbalance", "cputime", 0.01, fmt])
    out = _same(db, calls)
    assert any(o["status"] == 0 and o["call"][0] == "iterations" for o in out)
    assert any(o["status"] == 0 and o["call"][0] == "imbalance" and '"rows": [\n' in o["text"]
               for o in out if o["call"][-1] == JSON)


@pytest.mark.parametrize("rpn", [2, 10])
def test_ps_congestion_byte_identical(rpn):
    db = ref_db(scenarios.aurora(ranks_per_node=rpn, seed=2025))
    calls = []
    for fmt in (CSV, JSON):
        calls.append(["congestion", "MPI_*", "dbscan", 2, 0.0, fmt])
        calls.append(["congestion", "MPI_*", "kmeans", 2, 0.0, fmt])
        calls.append(["congestion", "MPI_Wait*", "dbscan", 2, 0.0, fmt])
        calls.append(["congestion", "NoSuchCall*", "dbscan", 2, 0.0, fmt])
    out = _same(db, calls)
    assert sum(o["status"] == 0 for o in out) >= 4

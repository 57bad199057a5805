"""GPU: the drop-in C++ binding (integration/perfslice_gpu.*) against the
UNMODIFIED reference through the reference's own types — tests/dropin/
dropin_test.cpp, built by tests/dropin/build.sh, prints one PASS/FAIL line per
case like the reference's acceptance suite."""
from __future__ import annotations

import os
import subprocess

import pytest

from tests.helpers import ROOT

pytestmark = pytest.mark.gpu

BIN = os.path.join(ROOT, "tests", "dropin", "_build", "dropin_test")


def test_dropin_binding_matches_reference():
    assert os.path.exists(BIN), f"{BIN} missing: run tests/dropin/build.sh where the reference exists"
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    fails = [ln for ln in r.stdout.splitlines() if ln.startswith("FAIL")]
    assert r.returncode == 0 and not fails, "\n".join(fails) or r.stderr
    assert sum(ln.startswith("PASS") for ln in r.stdout.splitlines()) >= 30

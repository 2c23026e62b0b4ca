"""GPU: the C++ drop-in headers (include/fastleg/*.hpp) over libfastleg_b200.

* acceptance_dropin -- the reference's own acceptance suite
  (proj/tests/acceptance.cpp, 10 criteria) compiled UNMODIFIED against our
  headers (tests/cpp/build.sh), run on the B200;
* roundtrip_dropin  -- the reference's demo (proj/demos/roundtrip.cpp);
* dropin_checks     -- our checks of error types, mutable plans, batching.
"""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
BIN = os.path.join(ROOT, "tests", "_bin")


def run(name, timeout=900):
    path = os.path.join(BIN, name)
    assert os.path.exists(path), f"{path} missing: run tests/cpp/build.sh (part of __graft_entry__.build())"
    p = subprocess.run([path], capture_output=True, text=True, timeout=timeout, cwd=BIN)
    print(p.stdout[-4000:])
    return p


def test_reference_acceptance_suite_on_gpu():
    p = run("acceptance_dropin")
    assert p.returncode == 0, p.stdout + p.stderr
    assert "all criteria passed" in p.stdout


def test_reference_roundtrip_demo_on_gpu():
    p = run("roundtrip_dropin")
    assert p.returncode == 0, p.stdout + p.stderr


def test_dropin_checks():
    p = run("dropin_checks")
    assert p.returncode == 0, p.stdout + p.stderr

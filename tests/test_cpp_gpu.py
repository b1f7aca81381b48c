"""Runs the C++ host-side parity program (tests/cpp/test_adapter.cpp: include/evb/evb.hpp +
evobench_adapter.hpp against the unmodified reference, built by __graft_entry__.build())."""
import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parent / "cpp" / "_build" / "test_adapter"

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not BIN.exists(), reason="C++ adapter test not built (needs /root/reference at build time)")
def test_cpp_adapter_against_reference():
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failure(s)" in r.stdout

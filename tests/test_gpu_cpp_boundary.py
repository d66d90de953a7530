"""GPU: the C++ façade (include/fastusp/uspsim_compat.hpp) driven by the same harness code
as the reference's own uspsim library, in one process (tests/cpp/compat_vs_reference.cpp)."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

BIN = os.path.join(os.path.dirname(__file__), "cpp", "_build", "compat_vs_reference")


def test_cpp_facade_matches_reference_library(cuda, fu):
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/_build not built (needs /root/reference at build time)")
    p = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    lines = [json.loads(x) for x in p.stdout.splitlines() if x.startswith("{")]
    bad = [x for x in lines if x.get("ok") is False]
    assert p.returncode == 0 and not bad, (bad, p.stderr[-2000:])
    assert any(x.get("check") == "usp_n8_r8_fp8" for x in lines)

"""GPU: the CLI's verify and simulate commands end to end."""
import json
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu


def cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_2602_10940_b200", *args],
                          capture_output=True, text=True, timeout=600)


def test_cli_verify_passes(cuda):
    p = cli("verify", "--workers", "4", "--max-ring", "2", "--dims", "1x8x512x128")
    assert p.returncode == 0, p.stderr
    rep = json.loads(p.stdout)
    assert rep["pass"] and rep["mesh"]
    names = [c["case"] for c in rep["cases"]]
    assert "e4m3_codec_roundtrip" in names and any(n.startswith("usp_N4_R2") for n in names)
    assert all(c["pass"] for c in rep["cases"])


def test_cli_simulate_reports_traffic_and_timeline(cuda):
    p = cli("simulate", "--workers", "4", "--max-ring", "2", "--dims", "1x8x512x128",
            "--pipelined", "--fp8-kv")
    assert p.returncode == 0, p.stderr
    rep = json.loads(p.stdout)
    assert rep["rel_l2_vs_single_gpu"] < 0.1
    ops = {e["op"] for e in rep["traffic"]}
    assert ops == {"all_to_all", "send"}
    assert rep["timeline"]

"""CPU: the cost model against SPEC's worked examples and the reference
fabric's traffic, and the CLI's cost command / exit-code contract."""
import csv
import io
import subprocess
import sys

import numpy as np
import pytest

from paper_2602_10940_b200 import costmodel as cm


def test_pipeline_timeline_spec_examples():
    t = cm.pipeline_timeline(2.0, 0.0, 4)       # comm = 0 -> equal, hidden 1
    assert t["serial_total"] == t["pipelined_total"] == 8.0 and t["hidden_fraction"] == 1.0
    t = cm.pipeline_timeline(2.0, 1.0, 4)
    assert t["serial_total"] == 11.0 and t["pipelined_total"] == 8.0 and t["hidden_fraction"] == 1.0
    t = cm.pipeline_timeline(2.0, 3.0, 4)
    assert t["serial_total"] == 17.0 and t["pipelined_total"] == 11.0
    assert abs(t["hidden_fraction"] - 2 / 3) < 1e-12


def test_volumes_match_reference_traffic():
    from oracle import ref, ref_available
    from oracle import restate as R
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    q, k, v = (R.rng_tensor(s, (1, 8, 32, 16)) for s in (1, 2, 3))
    w = cm.WorkloadProfile(B=1, H=8, S=32, D=16)
    for n, r in ((2, 1), (4, 2), (8, 4), (8, 8)):
        for fp8 in (False, True):
            _, a2a, snd = ref.usp_attention(q, k, v, n, r, fp8=fp8, traffic=True)
            u = n // r
            want = cm.comm_volume_ulysses(w, u, width=4, fp8=fp8, out_width=4, n=n)
            assert int(a2a[0]) == want
            assert int(snd[0]) == cm.comm_volume_ring(w, r, u, width=4, fp8=fp8)
    assert cm.comm_volume_ulysses(w, 1) == 0 and cm.comm_volume_ring(w, 1, 8) == 0
    # SPEC.md:390 example, per rank (the SPEC's 256 B is both ranks)
    assert cm.comm_volume_ulysses(cm.WorkloadProfile(B=1, H=2, S=8, D=4), 2, width=2) == 128
    # SPEC.md:395 example: its expression 2*(2*4*4*2)*1 evaluates to 128 (the "256" printed
    # there is an arithmetic slip; the reference fabric agrees with 128, checked above)
    assert cm.comm_volume_ring(cm.WorkloadProfile(B=1, H=2, S=8, D=4), 2, 1, width=2) == 128


def test_step_latency_properties():
    hw = cm.HardwareProfile()
    w = cm.WorkloadProfile()
    b = cm.step_latency(hw, w, 8, 2)
    assert abs(b.total - (b.compute + b.exposed_comm + b.launch)) < 1e-15
    # monotone in bandwidth and launch count
    slow = cm.step_latency(cm.HardwareProfile(link_bandwidth=hw.link_bandwidth / 2), w, 8, 2)
    assert slow.total >= b.total and slow.exposed_comm > b.exposed_comm
    more = cm.step_latency(hw, cm.WorkloadProfile(kernels_per_layer=50), 8, 2, compiled=False)
    assert more.total > cm.step_latency(hw, w, 8, 2, compiled=False).total
    # pipelined <= serial, equal at R = 1
    assert cm.step_latency(hw, w, 8, 4, pipelined=True).total <= \
        cm.step_latency(hw, w, 8, 4, pipelined=False).total
    assert cm.step_latency(hw, w, 8, 1, pipelined=True).total == \
        cm.step_latency(hw, w, 8, 1, pipelined=False).total
    rep = cm.speedup_report(cm.step_latency(hw, w, 1, 1, compiled=False),
                            cm.step_latency(hw, w, 1, 1, compiled=True))
    assert rep["speedup"] > 1.0
    with pytest.raises(ValueError):
        cm.step_latency(hw, cm.WorkloadProfile(H=3), 4, 1)


def test_cli_cost_csv_and_exit_codes():
    p = subprocess.run([sys.executable, "-m", "paper_2602_10940_b200", "cost", "--format", "csv",
                        "--dims", "1x24x4608x128"], capture_output=True, text=True, timeout=120)
    assert p.returncode == 0, p.stderr
    rows = list(csv.DictReader(io.StringIO(p.stdout)))
    assert rows and all(abs(float(r["total_ms"]) - (float(r["compute_ms"]) +
                                                    float(r["comm_exposed_ms"]) +
                                                    float(r["launch_ms"]))) < 1e-9 for r in rows)
    # infeasible mesh (H=3, N=4, max_ring=1) -> exit 2
    p = subprocess.run([sys.executable, "-m", "paper_2602_10940_b200", "verify", "--workers", "4",
                        "--max-ring", "1", "--dims", "1x3x64x128"], capture_output=True, text=True,
                       timeout=120)
    assert p.returncode == 2 and "invalid configuration" in p.stderr


def test_block_latency_peer_hides_input_alltoall():
    hw, w = cm.HardwareProfile(), cm.WorkloadProfile()
    one = cm.block_latency(hw, w, 1)
    assert one["exposed_comm_us"] == 0.0
    for n in (2, 4, 8):
        fused, nccl = cm.block_latency(hw, w, n, peer=True), cm.block_latency(hw, w, n, peer=False)
        # the QKV projection's epilogue carries the input all-to-all: what is left exposed is
        # the signal kernels and the last attention wave's output stores
        assert fused["exposed_comm_us"] < nccl["exposed_comm_us"]
        assert fused["total_us"] < one["total_us"]
        parts = fused["qkv_proj_us"] + fused["attention_us"] + fused["movers_us"] + \
            fused["exposed_comm_us"] + fused["out_proj_us"]
        assert abs(parts - fused["total_us"]) < 1e-6

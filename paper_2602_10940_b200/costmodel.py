"""Analytical cost model of the USP layer, calibrated to B200.

The reference specifies this model but ships no code for it.  Volumes follow SPEC.md's
closed forms (checked against the C ABI's traffic counters in tests); time terms use
B200 numbers measured in this repo (profiles/): attention throughput per per-rank shape,
NVLink 5 peer bandwidth, kernel launch overhead with and without CUDA-Graph replay.
"""
from __future__ import annotations

import json
import math
from dataclasses import asdict, dataclass, field
from typing import Dict, List, Optional


# per-rank attention launches of the BASELINE meshes, measured on one B200 (f16 output)
ATTN_MEASURED = {"24x4608": 1299.6, "12x4608": 1229.2, "6x4608": 1049.9, "3x4608": 877.4,
                 "12x4224": 1161.2, "6x3584": 889.5, "24x7168": 1142.6}  # profiles/r02_vmesh.jsonl, 3x4608: attn_kv2_kernel (r02_ab_kv2.jsonl)


# tcgen05 projection GEMMs of the FLUX block (C = 3072, H = 24) at per-rank token counts S/N,
# measured on one B200 (tools/cpp/proj_bench, profiles/r02_proj_tokens.jsonl):
# tokens -> (QKV projection incl. the QK RMSNorm + RoPE epilogue us, output projection us)
PROJ_MEASURED_US = {4608: (178.6, 53.0), 2304: (98.4, 37.0), 1152: (66.8, 20.6), 576: (39.7, 14.5)}


@dataclass
class HardwareProfile:
    """SPEC.md:373-376.  Defaults: one B200 on an NVSwitch node."""
    link_bandwidth: float = 770e9       # B/s per direction per GPU (measured peer copy)
    link_latency: float = 6e-6          # s per NCCL group call (launch + handshake)
    peer_signal: float = 2e-6           # s per peer-window signal-and-wait kernel (fused path)
    # per kernel launch, eager: calibrated on the 60-layer Qwen stack at world 1 (2 kernels a
    # layer; profiles/r02_vmesh.jsonl "cuda_graph_stack": 34.29 ms eager vs 33.40 ms replayed
    # = 14.8 us a layer), with graph_residual assumed (one measurement cannot separate them)
    launch_overhead: float = 7.8e-6
    graph_residual: float = 0.05        # fraction of launch cost left under graph replay
    element_width: int = 2              # bytes per Q/K/V element on the wire (bf16/f16)
    peak_tflops: float = 1618.9         # measured dense bf16 burst (MEASURED_PEAKS.json)
    attn_efficiency: float = 0.81       # fallback: attention-kernel fraction of peak at FLUX U=1
    # Measured attention-kernel throughput (TFLOP/s) per per-rank launch shape "heads x span"
    # (tools/virtual_mesh_bench.py, profiles/r02_vmesh.jsonl); attention_seconds interpolates it over
    # log(FLOP per launch) -- small per-rank launches run well below the U=1 efficiency.
    attn_tflops_measured: Dict[str, float] = field(default_factory=lambda: dict(ATTN_MEASURED))

    def __post_init__(self):
        for k, v in asdict(self).items():
            if isinstance(v, dict):
                continue
            if v <= 0:
                raise ValueError(f"HardwareProfile.{k} must be positive")

    def attn_tflops(self, flop: float) -> float:
        """Attention throughput at a launch of `flop` FLOP: piecewise-linear in log(FLOP)
        through the measured shapes (D = 128), clamped at the ends; the fallback efficiency
        when no measurements are loaded."""
        pts = []
        for key, tf in self.attn_tflops_measured.items():
            h, s = (int(x) for x in key.split("x"))
            pts.append((math.log(4.0 * h * s * s * 128), tf))
        if not pts:
            return self.peak_tflops * self.attn_efficiency
        pts.sort()
        x = math.log(max(flop, 1.0))
        if x <= pts[0][0]:
            return pts[0][1]
        if x >= pts[-1][0]:
            return pts[-1][1]
        for (x0, y0), (x1, y1) in zip(pts, pts[1:]):
            if x0 <= x <= x1:
                return y0 + (y1 - y0) * (x - x0) / (x1 - x0) if x1 > x0 else max(y0, y1)
        return pts[-1][1]


@dataclass
class WorkloadProfile:
    """SPEC.md:377-380."""
    B: int = 1
    H: int = 24
    S: int = 4608
    D: int = 128
    layers: int = 1
    kernels_per_layer: int = 2        # measured: V staging + attention at N=1 (bench gpu_launches)
    steps: int = 1
    other_compute_per_step: float = 0.0  # s, non-attention work (projections, MLP), if known


@dataclass
class LatencyBreakdown:
    """total == compute + exposed_comm + launch."""
    compute: float
    exposed_comm: float
    hidden_comm: float
    launch: float
    total: float = field(init=False)

    def __post_init__(self):
        self.total = self.compute + self.exposed_comm + self.launch

    def as_dict(self) -> Dict[str, float]:
        return {"compute_ms": self.compute * 1e3, "comm_exposed_ms": self.exposed_comm * 1e3,
                "comm_hidden_ms": self.hidden_comm * 1e3, "launch_ms": self.launch * 1e3,
                "total_ms": self.total * 1e3}


def comm_volume_ulysses(w: WorkloadProfile, u: int, width: int = 2, fp8: bool = False,
                        out_width: Optional[int] = None, n: Optional[int] = None) -> int:
    """Bytes one rank puts on the wire per layer for the two Ulysses all-to-alls: the
    reference fabric's TrafficLog closed form (equal to the C ABI counters).
    Local shards hold S/N rows (N = n, default U for a Ulysses-only mesh).  fp8: K and V
    travel as 1-byte codes plus one 4-byte scale each per destination.  (SPEC.md:390's
    worked example, 256 B for U=2,H=2,S=8,D=4,w=2, counts both ranks; one rank sends 128.)"""
    if u <= 1:
        return 0
    n_local = w.S // (n or u)
    blk = w.B * (w.H // u) * n_local * w.D
    ow = width if out_width is None else out_width
    kv = (blk + 4) if fp8 else blk * width
    return (u - 1) * (blk * width + 2 * kv) + (u - 1) * blk * ow


def comm_volume_ring(w: WorkloadProfile, r: int, u: int, width: int = 2, fp8: bool = False) -> int:
    """2 * B * (H/U) * (S/R) * D * width * (R-1); codes + scale with fp8."""
    if r <= 1:
        return 0
    chunk = w.B * (w.H // u) * (w.S // r) * w.D
    part = (chunk + 4) if fp8 else chunk * width
    return (r - 1) * 2 * part


def pipeline_timeline(compute: float, comm: float, r: int) -> Dict[str, float]:
    """SPEC.md:398-406 (Alg. 2)."""
    serial = r * compute + (r - 1) * comm
    pipelined = compute + (r - 1) * max(compute, comm) if r > 1 else compute
    if comm <= 0 or r <= 1:
        hidden = 1.0
    else:
        hidden = 1.0 - (pipelined - r * compute) / ((r - 1) * comm)
    return {"serial_total": serial, "pipelined_total": pipelined,
            "hidden_fraction": max(0.0, min(1.0, hidden))}


def attention_seconds(hw: HardwareProfile, b: int, heads: int, s_q: int, s_kv: int, d: int) -> float:
    flop = 4.0 * b * heads * s_q * s_kv * d
    return flop / (hw.attn_tflops(flop) * 1e12)


def attention_waves(hw: HardwareProfile, b: int, heads: int, s_q: int, sms: int = 148) -> float:
    """Waves of output tiles the per-rank attention launch stores: 256-row q-blocks on the
    persistent kernel, whole 128-row tiles on the KV-split kernel when they fit one wave."""
    tiles128 = b * heads * -(-s_q // 128)
    if tiles128 <= sms:
        return 1.0
    return b * heads * -(-s_q // 256) / sms


def step_latency(hw: HardwareProfile, w: WorkloadProfile, n: int, r: int, pipelined: bool = True,
                 compiled: bool = True, fp8: bool = False, peer: bool = False,
                 out_width: Optional[int] = None) -> LatencyBreakdown:
    """SPEC.md:407-414 per denoising step: attention compute split over the mesh, Ulysses
    all-to-alls exposed, ring transfers through pipeline_timeline, launch term.

    peer=True models the peer-memory transport (csrc/peer.cu): the input reshard is the pack
    kernel's own stores into the members' windows (its bytes at link bandwidth plus one
    signal kernel, no NCCL group call), and the output reshard is the attention epilogue's
    stores -- overlapped with the compute of later tiles except for the last wave's; the ring's
    rounds are copy-engine copies into the next member's window plus one signal kernel."""
    if n % r or w.H % (n // r) or w.S % n:
        raise ValueError(f"infeasible mesh N={n} R={r} for H={w.H}, S={w.S}")
    u = n // r
    hp, span = w.H // u, w.S // r
    step_compute = attention_seconds(hw, w.B, hp, span, span, w.D)  # one ring step per rank
    ow = hw.element_width if out_width is None else out_width
    if peer and u > 1:
        total = comm_volume_ulysses(w, u, hw.element_width, fp8, out_width=ow, n=n)
        out_b = (u - 1) * w.B * hp * (w.S // n) * w.D * ow
        waves = attention_waves(hw, w.B, hp, span)
        a2a = (total - out_b) / hw.link_bandwidth + hw.peer_signal
        a2a += out_b / hw.link_bandwidth / max(waves, 1.0) + hw.peer_signal
    else:
        a2a = comm_volume_ulysses(w, u, hw.element_width, fp8, out_width=ow, n=n) / hw.link_bandwidth
        a2a += (2 * hw.link_latency) if u > 1 else 0.0
    # ring round: the K / V chunk over the link, plus an NCCL group call -- or, on the peer
    # ring, a copy-engine copy into the next member's window and one signal kernel
    per_round_comm = (comm_volume_ring(w, r, u, hw.element_width, fp8) / max(r - 1, 1)
                      / hw.link_bandwidth + (hw.peer_signal if peer else hw.link_latency)) if r > 1 else 0.0
    tl = pipeline_timeline(step_compute, per_round_comm, r)
    ring_total = tl["pipelined_total"] if pipelined else tl["serial_total"]
    compute = r * step_compute
    ring_exposed = ring_total - compute
    ring_hidden = (r - 1) * per_round_comm - ring_exposed
    launches = w.kernels_per_layer + (4 if u > 1 else 0) + (2 * (r - 1) if r > 1 else 0)
    launch = launches * hw.launch_overhead * (hw.graph_residual if compiled else 1.0)
    per_layer = LatencyBreakdown(compute, a2a + ring_exposed, max(ring_hidden, 0.0), launch)
    L = w.layers
    return LatencyBreakdown(per_layer.compute * L + w.other_compute_per_step,
                            per_layer.exposed_comm * L, per_layer.hidden_comm * L,
                            per_layer.launch * L)


def block_latency(hw: HardwareProfile, w: WorkloadProfile, n: int, peer: bool = True,
                  movers_us: Optional[float] = None) -> Dict[str, float]:
    """The whole FLUX joint-attention block per rank at U = N, R = 1 (fusp_usp_block): QKV
    projection -> USP layer -> output projection, from the measured per-rank GEMM times
    (PROJ_MEASURED_US; the block's C and H are the table's) and step_latency's layer.

    peer=True models the fused producer (csrc/peer.cu + proj_sm100.cu): the QKV projection's
    epilogue stores Q, K, V into the members' windows as its tiles complete, so the input
    all-to-all costs only what the link cannot move while the GEMM runs (plus one signal
    kernel); the output all-to-all is the attention epilogue's stores (step_latency peer);
    the output projection reads O in place.  movers_us: the operand staging of V and its
    range decision at N = 1 (8.2 us, profiles/r02_launches.md), the unpack-stage of the
    received Q, K, V slots and its decision at N > 1 (~6 us, profiles/r02_movers.jsonl)."""
    if movers_us is None:
        movers_us = 8.2 if n == 1 else 6.0
    if w.S // n not in PROJ_MEASURED_US:
        raise ValueError(f"no projection measurement at {w.S // n} tokens")
    qkv_us, out_us = PROJ_MEASURED_US[w.S // n]
    u = n
    hp = w.H // u
    attn = attention_seconds(hw, w.B, hp, w.S, w.S, w.D)
    if u == 1:
        comm = 0.0
    else:
        blk = w.B * hp * (w.S // n) * w.D
        in_bytes = (u - 1) * 3 * blk * hw.element_width
        out_bytes = (u - 1) * blk * hw.element_width
        waves = attention_waves(hw, w.B, hp, w.S)
        if peer:
            comm = max(0.0, in_bytes / hw.link_bandwidth - qkv_us * 1e-6) + hw.peer_signal
            comm += out_bytes / hw.link_bandwidth / max(waves, 1.0) + hw.peer_signal
        else:
            comm = (in_bytes + out_bytes) / hw.link_bandwidth + 2 * hw.link_latency
    total = qkv_us * 1e-6 + attn + movers_us * 1e-6 + comm + out_us * 1e-6
    return {"n": n, "qkv_proj_us": qkv_us, "attention_us": attn * 1e6, "movers_us": movers_us,
            "exposed_comm_us": comm * 1e6, "out_proj_us": out_us, "total_us": total * 1e6}


def speedup_report(base: LatencyBreakdown, opt: LatencyBreakdown) -> Dict[str, float]:
    """total ratio and per-component attribution of the delta."""
    d = {"compute": base.compute - opt.compute, "exposed_comm": base.exposed_comm - opt.exposed_comm,
         "launch": base.launch - opt.launch}
    assert abs(sum(d.values()) - (base.total - opt.total)) < 1e-12
    return {"speedup": base.total / opt.total, **{f"delta_{k}_ms": v * 1e3 for k, v in d.items()}}


def sweep(hw: HardwareProfile, w: WorkloadProfile, ns=(1, 2, 4, 8), fp8: bool = False,
          compiled: bool = True) -> List[Dict]:
    rows = []
    for n in ns:
        for r in [x for x in range(1, n + 1) if n % x == 0]:
            if w.H % (n // r) or w.S % n:
                continue
            for pip in (False, True):
                b = step_latency(hw, w, n, r, pipelined=pip, compiled=compiled, fp8=fp8)
                comm = b.exposed_comm + b.hidden_comm
                rows.append({"config": f"N{n}_R{r}_U{n // r}_{'pipe' if pip else 'serial'}",
                             **b.as_dict(),
                             "comm_fraction": b.exposed_comm / b.total if b.total else 0.0,
                             "hidden_fraction": (b.hidden_comm / comm) if comm else 1.0})
    return rows


def load_profile(path: Optional[str]) -> HardwareProfile:
    if not path:
        return HardwareProfile()
    with open(path) as f:
        return HardwareProfile(**json.load(f))

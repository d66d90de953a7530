#!/usr/bin/env python
"""Benchmark: FLUX-shape USP joint-attention layer on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl fastusp|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (one rank per GPU, NCCL)

A step is one USP attention layer (Ulysses all-to-all -> ring attention -> Ulysses
all-to-all) over FLUX-shaped synthetic tensors, B=1 S=4608 H=24 D=128, bf16 in, f16 out,
U=N R=1 by default (BASELINE configs[1]); total work is fixed as N grows (strong scaling).
`value` = whole-job TFLOP/s = 4*B*H*S^2*D / (max over ranks of the device time per step).
L2 (126 MB) is flushed between timed steps outside the per-step events: a 256 MiB write, then a
256 MiB read, so the step starts with none of its inputs in L2 and no dirty flush lines left to
write back (a write-only flush leaves ~126 MB of dirty lines whose write-back the next step pays).

`--impl reference` times the reference's own CPU implementation (oracle/_ref, the
uspsim library compiled from the reference sources) on this host's cores instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FLUX-shape USP attention layer latency (us) & TFLOP/s at 1/2/4/8 B200"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def peaks():
    try:
        with open(PEAKS) as f:
            return json.load(f), "measured"
    except OSError:
        return FALLBACK_PEAKS, "fallback"


def layer_flop(b, h, s, d):
    return 4.0 * b * h * s * s * d


# ---------------------------------------------------------------------------- clocks
class NvmlClockSampler:
    """SM clock + throttle reasons sampled every ~2 ms via NVML during the timed region
    (the same fields as the profiling recipe's nvidia-smi clocks line)."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device: int):
        import pynvml
        self.nv = pynvml
        pynvml.nvmlInit()
        self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
        self.samples, self.reasons = [], 0
        self._stop = threading.Event()

    def start(self):
        def loop():
            while not self._stop.is_set():
                try:
                    self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                    self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except self.nv.NVMLError:
                    pass
                time.sleep(0.002)
        self._t = threading.Thread(target=loop, daemon=True)
        self._t.start()
        t0 = time.time()
        while not self.samples and time.time() - t0 < 2:
            time.sleep(0.001)

    def stop(self):
        self._stop.set()
        self._t.join()
        mx = self.nv.nvmlDeviceGetMaxClockInfo(self.h, self.nv.NVML_CLOCK_SM)
        names = sorted(n for bit, n in self.REASONS.items() if self.reasons & bit)
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": mx, "reasons": names, "samples": len(self.samples),
                "source": "nvml"}


def make_clock_sampler(device: int):
    try:
        return NvmlClockSampler(device)
    except Exception:  # noqa: BLE001 -- fall back to nvidia-smi
        return ClockSampler(device)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------- reference arm
REF_U = 2            # BASELINE configs[0]'s mesh: usp_attention at U=2, R=1 (two ranks)
REF_HEADS = 2        # FLUX heads per reference run (one per Ulysses rank)


def cpu_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count() or 1, "cpu_model": model}


def cpu_sample(seq: int, runs: int, d: int = 128):
    """The reference's own protocol: `runs` concurrent uspsim::usp_attention calls (oracle/_ref,
    compiled from the reference sources), each under run_protocol(2) at U=2 R=1 -- the default
    deterministic scheduler, which serialises a run's two ranks on one core -- on its own
    REF_HEADS FLUX heads truncated to `seq` tokens.  Returns (FLOP/s, wall seconds, FLOP)."""
    import numpy as np
    from oracle import ref
    rng = np.random.default_rng(7)
    data = [[rng.uniform(-1, 1, (1, REF_HEADS, seq, d)).astype(np.float32) for _ in range(3)]
            for _ in range(runs)]
    errs = []

    def one(x):
        try:
            ref.usp_attention(x[0], x[1], x[2], REF_U, 1)
        except Exception as e:  # noqa: BLE001 -- surfaced below
            errs.append(e)

    th = [threading.Thread(target=one, args=(x,)) for x in data]
    t0 = time.perf_counter()
    for t in th:
        t.start()
    for t in th:
        t.join()
    sec = time.perf_counter() - t0
    if errs:
        raise errs[0]
    flop = runs * layer_flop(1, REF_HEADS, seq, d)
    return flop / sec, sec, flop


def ref_runs():
    return max(1, min(os.cpu_count() or 1, 24 // REF_HEADS))


def ref_sample_desc(seq, runs):
    return (f"{runs} concurrent uspsim::usp_attention runs (oracle/_ref = the reference's C++), "
            f"each run_protocol(2) at U=2 R=1 with the deterministic scheduler (one core per run) "
            f"on {REF_HEADS} FLUX heads x {seq} tokens (S truncated from 4608; D=128)")


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    b, h, s, d = 1, 24, args.seq, 128
    runs, seq = ref_runs(), args.ref_seq
    for _ in range(args.warmup):
        cpu_sample(min(seq, 256), runs, d)  # warm-up: page in the library, spin up the cores
    rates, walls = [], []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r, sec, _ = cpu_sample(seq, runs, d)
        rates.append(r)
        walls.append(sec)
    wall = time.perf_counter() - t0
    rate = statistics.median(rates)
    full_ms = layer_flop(b, h, s, d) / rate * 1e3
    line = {
        "metric": METRIC, "impl": "reference", "value": rate / 1e12, "unit": "TFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.median(walls) * 1e3,  # what one step (the sample) took
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (uniform[-1,1])",
        "config": {"workload": f"FLUX joint attention layer B={b} S={s} H={h} D={d} (sampled: "
                               f"{runs} x {REF_HEADS} heads x {seq} tokens per step)",
                   "parallelism": f"{runs} concurrent reference runs (host cores)",
                   "wall_s": wall, "step_s_min": min(walls), "step_s_max": max(walls), **cpu_info()},
        "cpu_baseline": {"value": rate / 1e12, "unit": "TFLOP/s", "cores": runs, "kind": "reference",
                         "sample": ref_sample_desc(seq, runs)},
        "e2e": {"value": rate / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "extrapolated_full_layer_ms": full_ms,
        "extrapolated_note": "the full FLUX layer (24 heads, S=4608) at the measured FLOP rate on "
                             "these cores -- an extrapolation, not a measurement",
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------- fastusp arm
def run_fastusp(args):
    import torch
    import torch.distributed as dist

    import paper_2602_10940_b200 as fu

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:  # bound every device-side wait of the peer self-check (read once by the lib)
        os.environ.setdefault("FUSP_TIMEOUT_S", "30")
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE",
              file=sys.stderr)
    n = world
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if n > 1:
        from paper_2602_10940_b200 import dist as fdist
        dist.init_process_group("nccl", device_id=dev)
        uid = fdist.broadcast_bytes(fu.WorkerContext.nccl_unique_id() if rank == 0 else None)
        ctx = fu.WorkerContext.nccl(uid, n, rank, local)
    else:
        fab = fu.Fabric(1)
        ctx = fu.WorkerContext.local(fab, 0, local)

    b, h, s, d = 1, args.heads, args.seq, 128
    r = args.ring
    if n % r:
        raise SystemExit(f"ring {r} must divide {n}")
    mesh = fu.make_mesh(n, r)
    sl = s // n
    flop = layer_flop(b, h, s, d)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    q = torch.empty(b, h, sl, d, device=dev, dtype=torch.bfloat16).uniform_(-1, 1, generator=gen)
    k = torch.empty_like(q).uniform_(-1, 1, generator=gen)
    v = torch.empty_like(q).uniform_(-1, 1, generator=gen)
    out = torch.empty(b, h, sl, d, device=dev, dtype=torch.float16)
    opts = fu.CommOptions(fp8_kv=args.fp8, pipelined_ring=not args.serial,
                          out_dtype=torch.float16, check_finite=False)
    stream = torch.cuda.Stream(device=dev)
    transport = "nccl" if n > 1 else "local (world 1)"
    if n > 1 and args.peer != "off":
        with torch.cuda.stream(stream):
            transport = setup_peer(fu, ctx, dist, dev, q, k, v, mesh, opts, n, r, args)
    flush = torch.empty(256 * 1024 * 1024 // 4, device=dev, dtype=torch.float32)
    flush_rd = torch.ones(256 * 1024 * 1024 // 4, device=dev, dtype=torch.float32)

    def flush_l2(i):
        flush.fill_(float(i))  # evicts everything (leaves dirty lines) ...
        flush_rd.sum()         # ... whose write-back this read pays, outside the step events

    def barrier():
        if n > 1:
            dist.barrier()

    with torch.cuda.stream(stream):
        graph = None
        if args.graph:
            graph = fu.LayerGraph(ctx, q[None], k[None], v[None], out[None], mesh, opts, 1)

        def step():
            if graph is not None:
                graph.launch(stream)
            else:
                fu.usp_attention(ctx, q, k, v, mesh, opts)

        for _ in range(args.warmup):
            step()
        stream.synchronize()
        # ---- timed region: K layers, per-step CUDA events, L2 flushed between steps
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        clocks = make_clock_sampler(local)
        clocks.start()
        launches0 = fu.kernel_launch_count()
        barrier()
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush_l2(i)
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        stream.synchronize()
        barrier()
        torch.cuda.synchronize()
        launches = fu.kernel_launch_count() - launches0
        clk = clocks.stop()
        step_ms = [a.elapsed_time(z) for a, z in ev]
        t_ms = sum(step_ms) / len(step_ms)
        if n > 1:
            tt = torch.tensor([t_ms], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_ms = float(tt.item())
        # graph launches are counted by capture (kernels inside the graph): count per replay
        if graph is not None:
            per_layer = graph_kernel_count(fu, ctx, q, k, v, mesh, opts)
            launches = per_layer * args.steps

        # ---- dominant kernel alone (attention on resident bf16/f16 operands)
        att = attention_roofline(fu, dev, stream, b, h, s, d, n, args)
        # ---- the same kernel inside the layer: eager steps (L2 flushed between them), the
        # context's per-step CUDA events around each attention launch on the compute stream
        inl = []
        for i in range(args.steps):
            flush_l2(i)
            fu.usp_attention(ctx, q, k, v, mesh, opts)
            stream.synchronize()
            comp, _ = ctx.ring_timings()
            inl.append(sum(comp))
        att_us_layer = 1e3 * sum(inl) / len(inl) / r  # per attention launch (R per layer)
        # ---- ring hidden fraction when the mesh has a ring
        hidden = ring_hidden(fu, ctx, q, k, v, mesh, opts, stream) if r > 1 else None
        # ---- end to end through the reference-facing host-buffer call
        e2e = end_to_end(fu, ctx, q, k, v, mesh, opts, stream, flop, n, args)
    if graph is not None:
        graph.close()

    if rank == 0:
        pk, kind = peaks()
        flop_launch = flop / n / r  # one attention launch: this rank's heads x one ring chunk
        achieved = flop_launch / (att_us_layer * 1e-6) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": pk["bf16_tflops"],
                "unit": "TFLOP/s", "frac": achieved / pk["bf16_tflops"],
                "traffic": att.get("traffic"), "kernel": "attn_fwd_kernel",
                "peak_source": f"{kind} bf16 burst (MEASURED_PEAKS.json)",
                "algorithmic_flop_per_launch": flop_launch, "avg_launch_us": att_us_layer,
                "timing": "CUDA events around each attention launch inside eager layer steps "
                          "(compute stream, L2 flushed between steps)",
                "standalone_us": att["us"], "standalone_tflops": att["tflops"]}
        cpu = cpu_baseline(args)
        line = {
            "metric": METRIC, "value": flop / (t_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
            "n_gpus": n, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms,
            "latency_us": t_ms * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (uniform[-1,1])",
            "config": {"workload": f"FLUX joint attention layer B={b} S={s} H={h} D={d} "
                                   f"(4096 img + 512 txt tokens)",
                       "mesh": {"ulysses": n // r, "ring": r}, "parallelism": f"usp_u{n // r}_r{r}",
                       "fp8_kv": bool(args.fp8), "pipelined_ring": not args.serial,
                       "cuda_graph": bool(args.graph), "out_dtype": "f16",
                       "ulysses_transport": transport,
                       "l2": "flushed between steps (256 MiB write + 256 MiB read, outside the step events)",
                       "flop_per_layer": flop},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk,
        }
        if hidden is not None:
            line["ring"] = hidden
        print(json.dumps(line), flush=True)
    ctx.close()
    if n > 1:
        dist.destroy_process_group()
    return 0


def setup_peer(fu, ctx, dist, dev, q, k, v, mesh, opts, n, r, args):
    """Peer-memory Ulysses transport for N > 1 (fusp_ctx_peer_*): windows created locally,
    handles all-gathered over torch.distributed, mapped (CUDA IPC); then a self-check layer
    must match the NCCL layer bit for bit on every rank, else every rank falls back to NCCL.
    Returns the transport description for the JSON line."""
    import torch

    def agree(ok: bool) -> bool:
        t = torch.tensor([1 if ok else 0], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return bool(t.item())

    ref = fu.usp_attention(ctx, q, k, v, mesh, opts).clone()
    torch.cuda.current_stream().synchronize()
    why = ""
    try:
        wb = fu.peer_window_bytes(n, r, tuple(q.shape), q.dtype, opts)
        h = ctx.peer_window(wb)
        ok = True
    except Exception as e:  # noqa: BLE001 -- reported, NCCL stays the transport
        ok, why = False, f"window: {e}"
    if not agree(ok):
        return f"nccl (peer windows unavailable{': ' + why if why else ''})"
    handles = [None] * n
    dist.all_gather_object(handles, h)
    try:
        ctx.peer_open(handles)
        got = fu.usp_attention(ctx, q, k, v, mesh, opts).clone()
        ctx.synchronize()
        ok = torch.equal(got, ref) and ctx.peer_stats()[0] >= 1
        if not ok:
            why = "self-check mismatch"
    except Exception as e:  # noqa: BLE001
        ok, why = False, f"self-check: {e}"
    if agree(ok):
        return "peer-memory (pack / attention-epilogue stores into NVLink-mapped windows)"
    try:
        ctx.disable_peer_memory()
    except Exception:  # noqa: BLE001
        pass
    return f"nccl (peer path rejected: {why or 'another rank failed'})"


def graph_kernel_count(fu, ctx, q, k, v, mesh, opts):
    """fastusp kernels one eager layer launches (== the kernels inside one graph replay)."""
    import torch
    c0 = fu.kernel_launch_count()
    fu.usp_attention(ctx, q, k, v, mesh, opts)
    torch.cuda.current_stream().synchronize()
    return fu.kernel_launch_count() - c0


def attention_roofline(fu, dev, stream, b, h, s, d, n, args):
    """Average device time of the attention kernel alone on this rank's Ulysses shard
    (H/U heads x S rows), CUDA events on its launching stream."""
    import torch
    u = n // args.ring
    hp, span = h // u, s // args.ring
    q = torch.empty(b, hp, span, d, device=dev, dtype=torch.bfloat16).uniform_(-1, 1)
    kk = torch.empty_like(q).uniform_(-1, 1)
    vv = torch.empty(b, hp, span, d, device=dev, dtype=torch.float16).uniform_(-1, 1)
    for _ in range(3):
        fu.attention_with_lse(q, kk, vv, out_dtype=torch.float16)
    reps = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.current_stream().synchronize()
    e0.record()
    for _ in range(reps):
        fu.attention_with_lse(q, kk, vv, out_dtype=torch.float16)
    e1.record()
    e1.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    flop = layer_flop(b, hp, span, d)
    res = {"us": us, "flop": flop, "tflops": flop / (us * 1e-6) / 1e12}
    tp = os.path.join(ROOT, "profiles", "attention_traffic.json")
    if os.path.exists(tp):
        try:
            with open(tp) as f:
                t = json.load(f)
            key = f"h{hp}_s{span}"
            res["traffic"] = t.get(key)
        except (OSError, ValueError):
            pass
    return res


def ring_hidden(fu, ctx, q, k, v, mesh, opts, stream):
    """hidden = 1 - (t_pipe - R*t_step)/((R-1)*t_comm) from per-step events."""
    import dataclasses
    import torch
    ser = dataclasses.replace(opts, pipelined_ring=False)
    fu.usp_attention(ctx, q, k, v, mesh, ser)
    torch.cuda.current_stream().synchronize()
    comp, comm = ctx.ring_timings()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pip = dataclasses.replace(opts, pipelined_ring=True)
    e0.record()
    fu.usp_attention(ctx, q, k, v, mesh, pip)
    e1.record()
    e1.synchronize()
    r = len(comp)
    t_step = sum(comp) / r
    t_comm = sum(comm[1:]) / max(r - 1, 1)
    t_pipe = e0.elapsed_time(e1)
    hidden = 1.0 - (t_pipe - r * t_step) / ((r - 1) * t_comm) if t_comm > 0 else None
    return {"steps": r, "t_step_ms": t_step, "t_comm_ms": t_comm, "t_pipelined_layer_ms": t_pipe,
            "hidden_fraction": hidden}


def end_to_end(fu, ctx, q, k, v, mesh, opts, stream, flop, n, args):
    """Same metric through the host-buffer C-ABI call: pinned H2D of q,k,v, the layer,
    D2H of the output, all inside the timed region."""
    import torch
    hq, hk, hv = (t.cpu().pin_memory() for t in (q, k, v))
    hout = torch.empty(q.shape, dtype=opts.out_dtype).pin_memory()
    h2d = sum(t.numel() * t.element_size() for t in (hq, hk, hv))
    d2h = hout.numel() * hout.element_size()
    for _ in range(2):
        fu.usp_attention_host(ctx, hq, hk, hv, mesh, opts, out=hout)
    reps = max(3, min(args.steps, 10))
    t = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fu.usp_attention_host(ctx, hq, hk, hv, mesh, opts, out=hout)
        e1.record(stream)
        e1.synchronize()
        t.append(e0.elapsed_time(e1))
    ms = statistics.median(t)
    if n > 1:
        import torch.distributed as dist
        tt = torch.tensor([ms], device=q.device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    return {"value": flop / (ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": ms,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "path": "fusp_usp_attention_host (pinned host bf16 in, pinned host f16 out; H2D / layer / D2H "
                    "pipelined over head chunks)"}


def cpu_baseline(args):
    """The reference's CPU path on this host, rank 0 at N=1: the --impl reference sample, three
    times (median and range), with the host's core count and model."""
    if args.no_cpu_baseline:
        return None
    try:
        runs, seq = ref_runs(), args.ref_seq
        cpu_sample(256, runs)  # warm-up
        res = [cpu_sample(seq, runs) for _ in range(3)]
        rates = sorted(r for r, _, _ in res)
        return {"value": rates[1] / 1e12, "unit": "TFLOP/s", "cores": runs, "kind": "reference",
                "sample": ref_sample_desc(seq, runs) + "; median of 3",
                "range": [rates[0] / 1e12, rates[2] / 1e12],
                "seconds": [round(t, 3) for _, t, _ in res], **cpu_info()}
    except Exception as e:  # noqa: BLE001 -- the baseline is reported, never required
        return {"value": None, "unit": "TFLOP/s", "cores": 0, "kind": "reference",
                "sample": f"unavailable: {e}"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["fastusp", "reference"], default="fastusp")
    ap.add_argument("--seq", type=int, default=4608)
    ap.add_argument("--heads", type=int, default=24)
    ap.add_argument("--ring", type=int, default=1)
    ap.add_argument("--fp8", action="store_true")
    ap.add_argument("--serial", action="store_true", help="serial ring (default pipelined)")
    ap.add_argument("--no-graph", dest="graph", action="store_false")
    ap.add_argument("--ref-seq", type=int, default=1536,
                    help="tokens per head of the reference CPU sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--peer", choices=["auto", "off"], default="auto",
                    help="N > 1: Ulysses reshards through peer-memory windows (self-checked "
                         "against NCCL, falls back to it) or NCCL only")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_fastusp(args)


if __name__ == "__main__":
    sys.exit(main())

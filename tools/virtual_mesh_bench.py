#!/usr/bin/env python
"""Protocol measurements that need a mesh, on ONE B200: N ranks as threads over the
in-process fabric (copy-engine transfers), all sharing cuda:0.

Not a multi-GPU number (every rank shares the same SMs and HBM); it measures what a single
GPU can show about the mesh configurations of BASELINE.json:
  * per-rank attention kernel efficiency at each configuration's per-GPU shape;
  * the ring pipeline's hidden fraction from per-step CUDA events;
  * FP8 vs BF16 Ulysses all-to-all: bytes on the wire, layer time, accuracy;
  * CUDA-Graph replay vs eager launches for a stack of layers (launch overhead).
Prints one JSON object per measurement.
"""
from __future__ import annotations

import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2602_10940_b200 as fu  # noqa: E402


def flop(h, s, d=128, b=1):
    return 4.0 * b * h * s * s * d


def kernel_tflops(hp, span, reps=20):
    q = torch.empty(1, hp, span, 128, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1)
    k = torch.empty_like(q).uniform_(-1, 1)
    v = torch.empty(1, hp, span, 128, device="cuda", dtype=torch.float16).uniform_(-1, 1)
    for _ in range(3):
        fu.attention_with_lse(q, k, v, out_dtype=torch.float16)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fu.attention_with_lse(q, k, v, out_dtype=torch.float16)
    e1.record()
    e1.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    return {"shape": [1, hp, span, 128], "us": us, "tflops": flop(hp, span) / (us * 1e-6) / 1e12}


def mesh_layer(n, r, s, h=24, fp8=False, block=False, pipelined=True, steps=5):
    """Time one USP layer across n ranks sharing the GPU (max over ranks of per-rank events)."""
    sl = s // n
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    full = [torch.empty(1, h, s, 128, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1,
                                                                                    generator=g)
            for _ in range(3)]
    shards = [[t[:, :, i * sl:(i + 1) * sl].contiguous() for i in range(n)] for t in full]
    mesh = fu.make_mesh(n, r)
    opts = fu.CommOptions(fp8_kv=fp8, fp8_block=int(block), pipelined_ring=pipelined,
                          out_dtype=torch.float16, check_finite=False)

    def prog(ctx):
        k = ctx.rank()
        q, kk, v = shards[0][k], shards[1][k], shards[2][k]
        for _ in range(2):
            out = fu.usp_attention(ctx, q, kk, v, mesh, opts)
        torch.cuda.current_stream().synchronize()
        ts = []
        for _ in range(steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out = fu.usp_attention(ctx, q, kk, v, mesh, opts)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        comp, comm = ctx.ring_timings()
        return {"ms": statistics.median(ts), "out": out, "comp": comp, "comm": comm,
                "traffic": ctx.traffic()}

    rep = fu.run_protocol(n, prog)
    ms = max(x["ms"] for x in rep.results)
    out = torch.cat([x["out"].float() for x in rep.results], dim=2)
    res = {"n_ranks": n, "ulysses": n // r, "ring": r, "seq": s, "heads": h, "fp8_kv": fp8,
           "fp8_block": block, "pipelined": pipelined, "layer_ms_all_ranks_one_gpu": ms,
           "a2a_bytes_rank0": rep.results[0]["traffic"][0] // (steps + 2),
           "ring_bytes_rank0": rep.results[0]["traffic"][1] // (steps + 2)}
    comp, comm = rep.results[0]["comp"], rep.results[0]["comm"]
    if r > 1 and comp:
        res["ring_step_compute_ms"] = comp
        res["ring_step_comm_ms"] = comm
    return res, out, full


def main():
    torch.cuda.set_device(0)
    lines = []
    # per-rank kernel efficiency at each config's per-GPU attention shape
    for name, hp, span in (("flux_u1", 24, 4608), ("flux_u2", 12, 4608), ("flux_u4", 6, 4608),
                           ("flux_u8", 3, 4608), ("ring_u2r4_step", 12, 4224),
                           ("qwen_u4r2_step", 6, 3584)):
        r = kernel_tflops(hp, span)
        r["config"] = name
        lines.append({"measure": "attention_kernel_per_rank_shape", **r})
    # FP8 vs BF16 Ulysses at U=8 (BASELINE configs[3])
    base, out_bf16, full = mesh_layer(8, 1, 4608)
    f8, out_f8, _ = mesh_layer(8, 1, 4608, fp8=True)
    f8b, out_f8b, _ = mesh_layer(8, 1, 4608, fp8=True, block=True)
    ref = out_bf16
    for r_, o in ((base, out_bf16), (f8, out_f8), (f8b, out_f8b)):
        r_["rel_l2_vs_bf16_path"] = float((o - ref).norm() / ref.norm())
        lines.append({"measure": "usp_layer_virtual_mesh", **r_})
    # Ring-heavy mesh U=2 R=4, S=16896 (BASELINE configs[2]): serial vs pipelined
    for pip in (False, True):
        r_, _, _ = mesh_layer(8, 4, 16896, pipelined=pip, steps=3)
        if r_.get("ring_step_compute_ms"):
            c, m = r_["ring_step_compute_ms"], r_["ring_step_comm_ms"]
            r_["t_step_ms"] = sum(c) / len(c)
            r_["t_comm_ms"] = sum(m[1:]) / max(len(m) - 1, 1)
        lines.append({"measure": "usp_layer_virtual_mesh", **r_})
    ser = [x for x in lines if x.get("ring") == 4 and not x["pipelined"]][0]
    pip = [x for x in lines if x.get("ring") == 4 and x["pipelined"]][0]
    R = 4
    t_pipe = pip["layer_ms_all_ranks_one_gpu"]
    t_ser = ser["layer_ms_all_ranks_one_gpu"]
    lines.append({"measure": "ring_pipelining", "serial_ms": t_ser, "pipelined_ms": t_pipe,
                  "speedup": t_ser / t_pipe,
                  "note": "8 ranks share one GPU: compute steps of all ranks contend for the "
                          "same SMs, transfers are copy-engine D2D"})
    # CUDA graph vs eager: Qwen-Image-shaped stack (S=7168, H=24) on one GPU, U=1 R=1
    layers = 60
    s = 7168
    q = torch.empty(layers, 1, 24, s, 128, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1)
    k = torch.empty_like(q).uniform_(-1, 1)
    v = torch.empty_like(q).uniform_(-1, 1)
    out = torch.empty(layers, 1, 24, s, 128, device="cuda", dtype=torch.float16)
    mesh = fu.make_mesh(1, 1)
    opts = fu.CommOptions(out_dtype=torch.float16, check_finite=False)

    def prog(ctx):
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

        def eager():
            for i in range(layers):
                fu.usp_attention(ctx, q[i], k[i], v[i], mesh, opts)

        g = fu.LayerGraph(ctx, q, k, v, out, mesh, opts, layers=layers)
        res = {"eager": [], "graph": []}
        # alternate the two and take medians: the clock settles lower after the first
        # sustained ~30 ms, so whichever runs first would otherwise look faster
        for _ in range(3):
            for name, fn in (("eager", eager), ("graph", g.launch)):
                fn()
                st.synchronize()
                t0 = time.perf_counter()
                e0.record()
                fn()
                e1.record()
                e1.synchronize()
                res[name].append((e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3))
        g.close()
        med = lambda xs, i: statistics.median(x[i] for x in xs)  # noqa: E731
        return (med(res["eager"], 0), med(res["eager"], 1)), (med(res["graph"], 0), med(res["graph"], 1))

    eager, graph = fu.run_protocol(1, prog).results[0]
    lines.append({"measure": "cuda_graph_stack", "layers": layers, "seq": s, "heads": 24,
                  "eager_device_ms": eager[0], "eager_wall_ms": eager[1],
                  "graph_device_ms": graph[0], "graph_wall_ms": graph[1],
                  "stack_tflops_graph": layers * flop(24, s) / (graph[0] * 1e-3) / 1e12,
                  "timing": "median of 3 alternating eager / graph runs"})
    for x in lines:
        print(json.dumps(x), flush=True)


if __name__ == "__main__":
    main()

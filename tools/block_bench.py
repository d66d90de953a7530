"""The whole MMDiT joint-attention block through fusp_usp_block at FLUX / Qwen shapes on one
B200: QKV projection (+ QK RMSNorm / RoPE epilogue) -> USP layer -> output projection."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_10940_b200 as fu

for name, s in (("flux", 4608), ("qwen", 7168)):
    h, c = 24, 3072
    x = torch.empty(1, s, c, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1)
    wqkv = torch.empty(c, 3 * h * 128, device="cuda", dtype=torch.bfloat16).uniform_(-0.02, 0.02)
    wout = torch.empty(h * 128, c, device="cuda", dtype=torch.bfloat16).uniform_(-0.02, 0.02)
    cos, sin = fu.rope_tables(s)
    pro = fu.QKPrologue(q_norm_weight=torch.ones(128, device="cuda"), k_norm_weight=torch.ones(128, device="cuda"),
                        rope_cos=cos, rope_sin=sin)
    fab = fu.Fabric(1)
    ctx = fu.WorkerContext.local(fab, 0, 0)
    mesh = fu.make_mesh(1, 1)
    opts = fu.CommOptions(check_finite=False)
    for _ in range(3):
        fu.usp_block(ctx, x, wqkv, h, wout, mesh, pro, opts)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    reps = 10
    for _ in range(reps):
        fu.usp_block(ctx, x, wqkv, h, wout, mesh, pro, opts)
    e1.record(); e1.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    flop = 2.0 * s * c * 3 * h * 128 + 4.0 * h * s * s * 128 + 2.0 * s * h * 128 * c
    # the same blocks replayed from one CUDA graph (fusp_graph_capture_block), 4 layers per graph
    layers = 4
    xl = x.unsqueeze(0).repeat(layers, 1, 1, 1).contiguous()
    yl = torch.empty(layers, 1, s, c, device="cuda", dtype=torch.bfloat16)
    cs = torch.cuda.Stream()  # (capture needs a stream other than the legacy default one)
    with torch.cuda.stream(cs):
        g = fu.BlockGraph(ctx, xl, wqkv, h, wout, yl, mesh, prologue=pro, opts=opts, layers=layers)
        for _ in range(2):
            g.launch()
        torch.cuda.synchronize(); e0.record()
        for _ in range(reps):
            g.launch()
        e1.record(); e1.synchronize()
    ug = e0.elapsed_time(e1) * 1e3 / (reps * layers)
    g.close()
    print(json.dumps({"block": name, "tokens": s, "channels": c, "heads": h, "us": round(us, 1),
                      "graph_us": round(ug, 1), "flop": flop, "tflops": round(flop / us / 1e6, 1),
                      "graph_tflops": round(flop / ug / 1e6, 1)}), flush=True)
    ctx.close()

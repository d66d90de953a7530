"""Eager vs CUDA-graph timing of a 60-layer Qwen-shaped stack (S=7168, H=24, U=1 R=1), each
measured 3 times alternately, plus the graph over fresh-output-sized buffers reused per layer
(isolates output-traffic effects from graph effects)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_10940_b200 as fu

layers, s = int(os.environ.get("LAYERS", 60)), 7168
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
    res = []
    for rnd in range(3):
        for name, fn in (("eager", eager), ("graph", g.launch)):
            fn()
            st.synchronize()
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            res.append((name, round(e0.elapsed_time(e1), 3)))
    g.close()
    return res


print(fu.run_protocol(1, prog).results[0])

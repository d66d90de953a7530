"""Host-path (pinned H2D -> layer -> D2H, one C-ABI call) timing of the FLUX U=1 layer for
several head-chunk counts (FUSP_HOST_CHUNKS is read once per process, so each count runs in
its own process).  usage: python tools/e2e_probe.py"""
import os, statistics, subprocess, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if len(sys.argv) == 1:
    for n, hs in ((4, 1), (4, 2), (4, 3), (3, 3), (6, 3), (8, 3), (4, 1), (4, 3)):
        env = dict(os.environ, FUSP_HOST_CHUNKS=str(n), FUSP_HOST_H2D_STREAMS=str(hs))
        r = subprocess.run([sys.executable, __file__, "run"], env=env, capture_output=True, text=True)
        print(r.stdout.strip() or r.stderr[-400:])
    sys.exit(0)
import torch
import paper_2602_10940_b200 as fu
h, s, d = 24, 4608, 128
q, k, v = (torch.empty(1, h, s, d, dtype=torch.bfloat16).uniform_(-1, 1).pin_memory() for _ in range(3))
out = torch.empty(1, h, s, d, dtype=torch.float16).pin_memory()
ctx = fu.WorkerContext.local(fu.Fabric(1), 0, 0)
mesh = fu.make_mesh(1, 1)
opts = fu.CommOptions(out_dtype=torch.float16, check_finite=False)
for _ in range(3):
    fu.usp_attention_host(ctx, q, k, v, mesh, opts, out=out)
t = []
for _ in range(10):
    t0 = time.perf_counter()
    fu.usp_attention_host(ctx, q, k, v, mesh, opts, out=out)
    t.append((time.perf_counter() - t0) * 1e3)
ms = statistics.median(t)
print(f"chunks<={os.environ.get('FUSP_HOST_CHUNKS')} h2d streams {os.environ.get('FUSP_HOST_H2D_STREAMS')}: {ms:.3f} ms  {4 * h * s * s * d / ms / 1e9:.1f} TFLOP/s "
      f"(h2d {3 * q.numel() * 2 / 1e6:.1f} MB, d2h {out.numel() * 2 / 1e6:.1f} MB)")

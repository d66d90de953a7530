import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2602_10940_b200 as fu
from oracle import restate as R
from oracle.make_golden import qkv
def rl(a, b): return float(np.linalg.norm(a - b) / np.linalg.norm(b))
def run(q, k, v, n, r, **o):
    qs, ks, vs = ([torch.from_numpy(np.ascontiguousarray(s)).cuda().bfloat16() for s in R.split_sequence(x, n)] for x in (q, k, v))
    mesh = fu.make_mesh(n, r); opts = fu.CommOptions(**o)
    rep = fu.run_protocol(n, lambda ctx: fu.usp_attention(ctx, qs[ctx.rank()], ks[ctx.rank()], vs[ctx.rank()], mesh, opts))
    return torch.cat([x.float() for x in rep.results], 2).cpu().numpy()
for kf, vf in ((1, 1), (3, 1), (1, 37), (3, 37)):
    q, k, v = qkv((1, 8, 64, 128), (1, 8, 64, 128), seeds=(51, 52, 53)); k[:, 3] *= kf; v[:, 3] *= vf
    k = R.round_bf16(k); v = R.round_bf16(v)
    pb = R.usp_attention(q, k, v, 2, 1, fp8=True, per_block=True); pt = R.usp_attention(q, k, v, 2, 1, fp8=True)
    gb = run(q, k, v, 2, 1, fp8_kv=True, fp8_block=1); gt = run(q, k, v, 2, 1, fp8_kv=True)
    print(kf, vf, "gpu_pb-vs-pb", rl(gb, pb), "gpu_pt-vs-pt", rl(gt, pt), "gpu_pb-vs-gpu_pt", rl(gb, gt), "per-head", [round(rl(gb[:, h], pb[:, h]), 5) for h in range(8)])

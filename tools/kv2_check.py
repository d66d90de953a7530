"""Correctness + timing of the KV-split attention kernel (schedule "kv2") against the default
schedule and the fp64 oracle on a few shapes (ragged rows, odd KV tile counts)."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2602_10940_b200 as fu
from oracle import restate as R

def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))

for heads, sq, skv in [(3, 512, 640), (2, 200, 300), (3, 4608, 4608), (1, 128, 128), (2, 384, 1000), (5, 256, 129), (6, 4608, 4608), (24, 4608, 4608), (3, 4224, 4224)]:
    g = torch.Generator().manual_seed(heads * 7 + sq)
    q = torch.empty(1, heads, sq, 128).uniform_(-1, 1, generator=g).bfloat16()
    k = torch.empty(1, heads, skv, 128).uniform_(-1, 1, generator=g).bfloat16()
    v = torch.empty(1, heads, skv, 128).uniform_(-1, 1, generator=g).bfloat16()
    acc = {}
    for mode in ("auto", "kv2", "kv2split"):
        with fu.attention_schedule(mode):
            r = fu.attention_with_lse(q.cuda(), k.cuda(), v.cuda())
        torch.cuda.synchronize()
        acc[mode] = (r.out.cpu().numpy(), r.lse.cpu().numpy())
    rows = slice(0, min(sq, 256))
    wo, wl = R.attention_with_lse(q[:, :, rows].float().numpy(), k.float().numpy(), v.float().numpy())
    for mode, (o, l) in acc.items():
        print(json.dumps({"shape": [heads, sq, skv], "mode": mode, "rel_l2": rel(o[:, :, rows], wo),
                          "lse_max": float(np.abs(l[:, :, rows] - wl).max())}), flush=True)

"""Per-CTA segment timeline of one attn_kv2_kernel launch (trace build: tools/build_variants.sh
trace:-DFUSP_TRACE_BUILD=1, then FUSP_VARIANT=trace).  Events are SM cycles from each CTA's start.
usage: FUSP_VARIANT=trace python tools/attn_trace_kv2.py HEADS SEQ MODE [MAX_CTAS]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2602_10940_b200 as fu
from paper_2602_10940_b200._lib import lib
hp, s, mode = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
ctas = int(sys.argv[4]) if len(sys.argv) > 4 else 0
L = lib()
q = torch.empty(1, hp, s, 128, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1)
k = torch.empty_like(q).uniform_(-1, 1); v = torch.empty(1, hp, s, 128, device="cuda", dtype=torch.float16).uniform_(-1, 1)
SLOTS = 72 + 2 * 64 * 2
with fu.attention_schedule(mode, ctas):
    for _ in range(3): fu.attention_with_lse(q, k, v, out_dtype=torch.float16)
    L.fusp_attention_trace(1, None, 0)
    fu.attention_with_lse(q, k, v, out_dtype=torch.float16); torch.cuda.synchronize()
    buf = np.zeros(160 * SLOTS, np.uint64)
    L.fusp_attention_trace(0, buf.ctypes.data, buf.size)
GHZ = float(os.environ.get("GHZ", "1.9"))
tr = buf.reshape(160, SLOTS).astype(np.int64)
cs = [c for c in range(160) if tr[c, 0]]
us = lambda x: x / (GHZ * 1e3)
names = ["S0", "loop", "mlx", "pub", "merge0", "merged", "end"]
ends = []
for c in cs:
    b = tr[c, 0]
    row = [f"cta {c:3d} end {us(tr[c,1]-b):6.1f}"]
    ends.append(us(tr[c, 1] - b))
    for sg in range(8):
        ev = tr[c, 2 + 8 * sg: 2 + 8 * sg + 7]
        if not ev.any():
            break
        row.append(" | " + " ".join(f"{n}={us(e-b):.1f}" for n, e in zip(names, ev) if e))
    if c < 12 or c % 20 == 0 or c == cs[-1]:
        print("".join(row))
ends.sort()
print(f"{len(cs)} CTAs; end min {ends[0]:.1f} median {ends[len(ends)//2]:.1f} max {ends[-1]:.1f} us (at {GHZ} GHz)")

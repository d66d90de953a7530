"""Per-CTA timeline of one attention launch (debug globaltimer events, fusp_attention_trace).
usage: python tools/attn_trace.py HEADS SEQ [mode]"""
import ctypes, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2602_10940_b200 as fu
from paper_2602_10940_b200._lib import lib
hp, s = int(sys.argv[1]), int(sys.argv[2]); mode = sys.argv[3] if len(sys.argv) > 3 else "auto"
L = lib()
q = torch.empty(1, hp, s, 128, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1)
k = torch.empty_like(q).uniform_(-1, 1); v = torch.empty(1, hp, s, 128, device="cuda", dtype=torch.float16).uniform_(-1, 1)
with fu.attention_schedule(mode, 0):
    for _ in range(3): fu.attention_with_lse(q, k, v, out_dtype=torch.float16)
    L.fusp_attention_trace(1, None, 0)
    fu.attention_with_lse(q, k, v, out_dtype=torch.float16); torch.cuda.synchronize()
    buf = np.zeros(160 * 72, np.uint64)
    L.fusp_attention_trace(0, buf.ctypes.data, buf.size)
GHZ = float(os.environ.get("GHZ", "1.9"))  # events are SM cycles; per-CTA times from its own start
tr = buf.reshape(160, 72).astype(np.int64)
ctas = [c for c in range(160) if tr[c, 0]]
for c in ctas:
    base = tr[c, 0]
    tr[c][tr[c] != 0] -= base
t0 = 0
us = lambda x: x / (GHZ * 1e3)
print(f"{len(ctas)} CTAs; longest CTA {us(max(max(tr[c,1], tr[c,70]) for c in ctas)):.1f} us (at {GHZ} GHz)")
# thread 0's clock read can run ahead of a deferred-blocking bar.sync: the CTA end is
# the later of the two end stamps (slot 70 = softmax warp 4 after the same barrier)
ends = sorted(us(max(tr[c, 1], tr[c, 70])) for c in ctas)
print(f"CTA end: min {ends[0]:.1f} median {ends[len(ends)//2]:.1f} max {ends[-1]:.1f}")
agg = {"first_S": [], "compute": [], "epilogue": [], "gap": []}
for c in ctas[: int(os.environ.get("SHOW", "6"))]:
    line = [f"cta{c:3d} start {us(tr[c,0]):6.1f}"]
    for sgi in range(8):
        for t in range(2):
            b = 2 + (sgi * 2 + t) * 4
            if tr[c, b] == 0: continue
            e = [us(x) for x in tr[c, b:b + 4]]
            line.append(f"s{sgi}t{t}[{e[0]:.1f} S{e[1]:.1f} O{e[2]:.1f} E{e[3]:.1f}]")
    line.append(f"end {us(tr[c,1]):.1f} end(w4) {us(tr[c,70]):.1f}")
    print(" ".join(line))
for c in ctas:
    prev_end = None
    for sgi in range(8):
        b = 2 + (sgi * 2) * 4
        if tr[c, b] == 0: continue
        e = tr[c, b:b + 4] / (GHZ * 1e3)
        agg["first_S"].append(e[1] - e[0]); agg["compute"].append(e[2] - e[1]); agg["epilogue"].append(e[3] - e[2])
for k2, vals in agg.items():
    if vals: print(f"{k2:9s} n={len(vals)} median {statistics.median(vals):.2f} us  max {max(vals):.2f} us  sum/CTA {sum(vals)/len(ctas):.2f} us")

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
    buf = np.zeros(160 * 328, np.uint64)
    L.fusp_attention_trace(0, buf.ctypes.data, buf.size)
GHZ = float(os.environ.get("GHZ", "1.9"))  # events are SM cycles; per-CTA times from its own start
tr = buf.reshape(160, 328).astype(np.int64)
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
NAMES = ["start", "S", "O", "fin", "pub", "ml", "merged", "E"]
agg = {k: [] for k in ("first_S", "compute", "publish", "fin_wait", "gather", "merge", "final_store")}
for c in ctas[: int(os.environ.get("SHOW", "6"))]:
    line = [f"cta{c:3d}"]
    for sgi in range(4):
        for t in range(2):
            b = 2 + (sgi * 2 + t) * 8
            if tr[c, b] == 0 and sgi > 0: continue
            e = tr[c, b:b + 8]
            line.append(f"s{sgi}t{t}[" + " ".join(f"{n}{us(x):.1f}" for n, x in zip(NAMES, e) if x) + "]")
    line.append(f"end {us(max(tr[c,1], tr[c,70])):.1f}")
    print(" ".join(line))
for c in ctas:
    for sgi in range(4):
        b = 2 + (sgi * 2) * 8
        if tr[c, b + 2] == 0: continue
        e = tr[c, b:b + 8] / (GHZ * 1e3)
        agg["first_S"].append(e[1] - e[0]); agg["compute"].append(e[2] - e[1])
        if e[4]: agg["publish"].append(e[4] - e[2])
        if e[3]: agg["fin_wait"].append(e[3] - (e[4] if e[4] else e[2]))
        if e[5] and e[3]: agg["gather"].append(e[5] - e[3])
        if e[6] and e[5]: agg["merge"].append(e[6] - e[5])
        agg["final_store"].append(e[7] - (e[6] if e[6] else e[2]))
for k2, vals in agg.items():
    if vals: print(f"{k2:11s} n={len(vals)} median {statistics.median(vals):.2f} us  max {max(vals):.2f} us")

# steady-state KV steps of the first segment: softmax time (S ready -> P published) and the
# MMA chain (P published -> next S ready), per Q tile, medians over CTAs
for t in range(2):
    sm_t, chain = [], []
    for c in ctas:
        ev = tr[c, 72 + t * 128: 72 + t * 128 + 128].reshape(64, 2)
        n = int((ev[:, 0] != 0).sum())
        for j in range(2, n - 1):
            sm_t.append((ev[j, 1] - ev[j, 0]) / (GHZ * 1e3))
            chain.append((ev[j + 1, 0] - ev[j, 1]) / (GHZ * 1e3))
    if sm_t:
        print(f"tile {t}: softmax per KV step median {statistics.median(sm_t)*1e3:.0f} ns, "
              f"P->next S median {statistics.median(chain)*1e3:.0f} ns  (steps {len(sm_t)})")

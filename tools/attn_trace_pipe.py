"""Per-step pipeline timing of the attention kernel from its clock64 trace (first segment of
every CTA): softmax = S ready -> P published, chain = P published -> next S ready, period and
the phase offset between the two Q tiles.
usage: [FUSP_VARIANT=x] python tools/attn_trace_pipe.py [heads] [seq]"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2602_10940_b200 as fu
from paper_2602_10940_b200._lib import lib

hp = int(sys.argv[1]) if len(sys.argv) > 1 else 24
s = int(sys.argv[2]) if len(sys.argv) > 2 else 4608
L = lib()
q = torch.empty(1, hp, s, 128, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1)
k = torch.empty_like(q).uniform_(-1, 1)
v = torch.empty(1, hp, s, 128, device="cuda", dtype=torch.float16).uniform_(-1, 1)
SLOTS = 72 + 2 * 64 * 2
with fu.attention_schedule("whole", 0):
    for _ in range(3):
        fu.attention_with_lse(q, k, v, out_dtype=torch.float16)
    L.fusp_attention_trace(1, None, 0)
    fu.attention_with_lse(q, k, v, out_dtype=torch.float16)
    torch.cuda.synchronize()
    buf = np.zeros(160 * SLOTS, np.uint64)
    L.fusp_attention_trace(0, buf.ctypes.data, buf.size)
    L.fusp_attention_trace(0, None, 0)
tr = buf.reshape(160, SLOTS).astype(np.int64)
d = {n: [] for n in ("softmax", "chain", "period", "offset")}
for c in range(148):
    ev = tr[c, 72:].reshape(2, 64, 2)  # [tile][step][S ready, P published]
    for j in range(2, 62):
        if ev[0, j + 1, 0] == 0 or ev[1, j + 1, 0] == 0:
            break
        for t in range(2):
            d["softmax"].append(ev[t, j, 1] - ev[t, j, 0])
            d["chain"].append(ev[t, j + 1, 0] - ev[t, j, 1])
            d["period"].append(ev[t, j + 1, 0] - ev[t, j, 0])
        d["offset"].append(ev[1, j, 0] - ev[0, j, 0])
for n, v in d.items():
    print(f"{os.environ.get('FUSP_VARIANT', 'main'):5s} {n:8s} median {statistics.median(v):7.0f} cycles  "
          f"p10 {np.percentile(v, 10):7.0f}  p90 {np.percentile(v, 90):7.0f}  (n={len(v)})")
# whole-CTA view: total cycles, and per segment (tile 0): wait for the first S, KV loop, epilogue
seg = {n: [] for n in ("total", "first_S", "kv_loop", "epilogue", "gap_to_next")}
for c in range(148):
    seg["total"].append(tr[c, 70] - tr[c, 0])
    for ns in range(3):
        b = 2 + (ns * 2 + 0) * 8
        if tr[c, b] == 0 or tr[c, b + 7] == 0:
            continue
        seg["first_S"].append(tr[c, b + 1] - tr[c, b])
        seg["kv_loop"].append(tr[c, b + 2] - tr[c, b + 1])
        seg["epilogue"].append(tr[c, b + 7] - tr[c, b + 2])
        nb = 2 + ((ns + 1) * 2) * 8
        if ns < 2 and tr[c, nb + 1] != 0:
            seg["gap_to_next"].append(tr[c, nb + 1] - tr[c, b + 7])
for n, v in seg.items():
    if v:
        print(f"{os.environ.get('FUSP_VARIANT', 'main'):5s} {n:11s} median {statistics.median(v):8.0f} cycles  "
              f"p10 {np.percentile(v, 10):8.0f}  p90 {np.percentile(v, 90):8.0f}  (n={len(v)})")
# FUSP_TRACE_EPI builds: epilogue sub-steps (o_done -> first O chunk -> all chunks -> barrier -> store read)
if os.environ.get("EPI"):
    sub = {n: [] for n in ("o_ld0", "chunks", "bar", "store_rd", "after")}
    for c in range(148):
        for ns in range(3):
            b = 2 + (ns * 2 + 0) * 8
            e = tr[c, b + 2:b + 8]
            if tr[c, b + 7] == 0 or e[1] == 0:
                continue
            sub["o_ld0"].append(e[1] - e[0]); sub["chunks"].append(e[2] - e[1])
            if e[3]:
                sub["bar"].append(e[3] - e[2])
            if e[4]:
                sub["store_rd"].append(e[4] - e[3]); sub["after"].append(e[5] - e[4])
    for n, v in sub.items():
        if v:
            print(f"epi {n:9s} median {statistics.median(v):8.0f}  p90 {np.percentile(v, 90):8.0f}")

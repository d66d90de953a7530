import ctypes, os, statistics, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2602_10940_b200 as fu
from paper_2602_10940_b200._lib import lib
hp, s = 24, 4608
L = lib()
q = torch.empty(1, hp, s, 128, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1)
k = torch.empty_like(q).uniform_(-1, 1); v = torch.empty(1, hp, s, 128, device="cuda", dtype=torch.float16).uniform_(-1, 1)
with fu.attention_schedule("whole", 0):
    for _ in range(3): fu.attention_with_lse(q, k, v, out_dtype=torch.float16)
    L.fusp_attention_trace(1, None, 0)
    fu.attention_with_lse(q, k, v, out_dtype=torch.float16); torch.cuda.synchronize()
    buf = np.zeros(160 * 328, np.uint64)
    L.fusp_attention_trace(0, buf.ctypes.data, buf.size)
tr = buf.reshape(160, 328).astype(np.int64)
d = {n: [] for n in ("ld", "max", "exp", "tail", "chain")}
for c in range(148):
    ev = tr[c, 72:72 + 5 * 48].reshape(48, 5)
    for j in range(2, 47):
        if ev[j + 1, 0] == 0: break
        d["ld"].append(ev[j, 1] - ev[j, 0]); d["max"].append(ev[j, 2] - ev[j, 1])
        d["exp"].append(ev[j, 3] - ev[j, 2]); d["tail"].append(ev[j, 4] - ev[j, 3])
        d["chain"].append(ev[j + 1, 0] - ev[j, 4])
for n, v in d.items():
    print(f"{n:6s} median {statistics.median(v):7.0f} cycles  p10 {np.percentile(v,10):7.0f}  p90 {np.percentile(v,90):7.0f}")

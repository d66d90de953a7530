"""Quick attention check under each schedule (one small shape), for kernel bring-up."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2602_10940_b200 as fu
from oracle import restate as R
from oracle.make_golden import qkv
h, sq, skv = (int(x) for x in sys.argv[2:5]) if len(sys.argv) > 4 else (1, 256, 1024)
mode = sys.argv[1] if len(sys.argv) > 1 else "whole"
q, k, v = qkv((1, h, sq, 128), (1, h, skv, 128))
ro, rl = R.attention_with_lse(q, k, v)
with fu.attention_schedule(mode, int(os.environ.get("CTAS", "0"))):
    r = fu.attention_with_lse(*(torch.from_numpy(x).cuda().bfloat16() for x in (q, k, v)))
    torch.cuda.synchronize()
o = r.out.cpu().numpy()
print(mode, h, sq, skv, "rel", np.linalg.norm(o - ro) / np.linalg.norm(ro), "dlse", np.abs(r.lse.cpu().numpy() - rl).max(), flush=True)

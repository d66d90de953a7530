"""One attention launch (after warm-up) at a named per-rank shape, for ncu captures.
usage: FUSP_VARIANT=... python tools/attn_once.py HEADS SEQ [mode]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_10940_b200 as fu
hp, s = int(sys.argv[1]), int(sys.argv[2])
mode = sys.argv[3] if len(sys.argv) > 3 else "auto"
q = torch.empty(1, hp, s, 128, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1)
k = torch.empty_like(q).uniform_(-1, 1)
v = torch.empty(1, hp, s, 128, device="cuda", dtype=torch.float16).uniform_(-1, 1)
with fu.attention_schedule(mode, 0):
    for _ in range(4):
        fu.attention_with_lse(q, k, v, out_dtype=torch.float16)
torch.cuda.synchronize()

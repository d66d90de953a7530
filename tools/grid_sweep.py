"""Stream-K grid size sweep for the small per-rank shapes (FLUX U=4/U=8, Qwen U=4 R=2 step):
median of 20 launches per grid cap.  usage: python tools/grid_sweep.py"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_10940_b200 as fu

for name, hp, s in (("flux_u8", 3, 4608), ("flux_u4", 6, 4608), ("qwen_u4r2_step", 6, 3584), ("flux_u2", 12, 4608)):
    q = torch.empty(1, hp, s, 128, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1)
    k = torch.empty_like(q).uniform_(-1, 1)
    v = torch.empty(1, hp, s, 128, device="cuda", dtype=torch.float16).uniform_(-1, 1)
    res = {}
    for rnd in range(3):
        for ctas in (0, 140, 128, 120, 108, 96, 74):
            with fu.attention_schedule("auto", ctas):
                for _ in range(3):
                    fu.attention_with_lse(q, k, v, out_dtype=torch.float16)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(20):
                    fu.attention_with_lse(q, k, v, out_dtype=torch.float16)
                e1.record()
                e1.synchronize()
                res.setdefault(ctas, []).append(e0.elapsed_time(e1) * 50.0)
    print(name, {c: round(statistics.median(t), 1) for c, t in res.items()}, flush=True)

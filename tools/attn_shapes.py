"""Attention kernel TFLOP/s at the per-rank shapes of the BASELINE configs (one GPU), under
each work schedule (whole q-blocks / stream-K split / auto)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_10940_b200 as fu

SHAPES = [("flux_u1", 24, 4608), ("flux_u2", 12, 4608), ("flux_u4", 6, 4608), ("flux_u8", 3, 4608),
          ("ring_u2r4_step", 12, 4224), ("qwen_u4r2_step", 6, 3584), ("qwen_u1", 24, 7168)]
MODES = sys.argv[1].split(",") if len(sys.argv) > 1 else ["whole", "split", "auto"]


def run(hp, span, reps=20):
    q = torch.empty(1, hp, span, 128, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1)
    k = torch.empty_like(q).uniform_(-1, 1)
    v = torch.empty(1, hp, span, 128, device="cuda", dtype=torch.float16).uniform_(-1, 1)
    for _ in range(3):
        fu.attention_with_lse(q, k, v, out_dtype=torch.float16)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(reps):
        fu.attention_with_lse(q, k, v, out_dtype=torch.float16)
    e1.record(); e1.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    return us, 4.0 * hp * span * span * 128 / (us * 1e-6) / 1e12


sel = os.environ.get("ATTN_SHAPES")  # comma-separated config names (default: all)
if sel:
    SHAPES = [x for x in SHAPES if x[0] in sel.split(",")]
for name, hp, span in SHAPES:
    for mode in MODES:
        with fu.attention_schedule(mode, 0):
            us, tf = run(hp, span)
        print(json.dumps({"config": name, "schedule": mode, "shape": [1, hp, span, 128],
                          "us": round(us, 1), "tflops": round(tf, 1)}), flush=True)

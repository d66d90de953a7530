"""Output-projection GEMM (fusp_out_projection) vs cuBLAS (torch.matmul on a token-major copy
of the same operands) at the BASELINE per-rank shapes; CUDA events, back-to-back reps."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_10940_b200 as fu


def timeit(f, reps=20):
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(reps):
        f()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


for name, h, s in (("flux_u1", 24, 4608), ("flux_u2", 24, 2304), ("flux_u8", 24, 576), ("qwen_u1", 24, 7168)):
    n = h * 128
    o = torch.empty(1, h, s, 128, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1)
    w = torch.empty(h * 128, n, device="cuda", dtype=torch.bfloat16).uniform_(-0.02, 0.02)
    a = o[0].transpose(0, 1).reshape(s, h * 128).contiguous()
    flop = 2.0 * s * h * 128 * n
    us = timeit(lambda: fu.out_projection(o, w, out_dtype=torch.bfloat16))
    ub = timeit(lambda: torch.matmul(a, w))
    print(json.dumps({"config": name, "m": s, "k": h * 128, "n": n, "fastusp_us": round(us, 1),
                      "fastusp_tflops": round(flop / us / 1e6, 1), "cublas_us_pretransposed": round(ub, 1),
                      "cublas_tflops": round(flop / ub / 1e6, 1)}), flush=True)

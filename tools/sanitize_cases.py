"""Small invocations of every fastusp kernel family for compute-sanitizer (memcheck /
racecheck / synccheck / initcheck): the attention kernel in both schedules (whole q-blocks and
stream-K split with its cross-CTA ticket merge), ring-step merges, the range-guarded staging
(common and rare path), the FP8 movers, and a 4-rank pipelined FP8 USP layer over the
in-process fabric.  Shapes are small: the sanitizer serialises and instruments every access.
usage: compute-sanitizer --tool memcheck python tools/sanitize_cases.py [case ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2602_10940_b200 as fu  # noqa: E402


def attention():
    q = torch.randn(1, 3, 640, 128, device="cuda", dtype=torch.bfloat16)
    k, v = torch.randn_like(q), torch.randn_like(q).half()
    for mode in ("whole", "split", "kv2", "kv2split"):
        with fu.attention_schedule(mode):
            fu.attention_with_lse(q, k, v, out_dtype=torch.float16)
    torch.cuda.synchronize()
    print("attention whole+split+kv2+kv2split ok", flush=True)


def staging():
    x = torch.randn(4, 384, 128, device="cuda")
    fu.stage_f16(x)                 # common path (in range)
    fu.stage_f16(x * 1e6)           # rare path: every head rewritten
    fu.stage_f16(x.bfloat16() * 1e-7)
    torch.cuda.synchronize()
    print("staging ok", flush=True)


def fp8_movers():
    x = torch.randn(1, 4, 256, 128, device="cuda")
    qt = fu.quantize(x)
    fu.dequantize(qt)
    codes, scales = fu.quantize_blocks(x, 256 * 128)
    fu.dequantize_blocks(codes, scales, 256 * 128)
    fu.requantize(qt.codes.flatten(), torch.ones(8, device="cuda"), qt.codes.numel() // 8)
    torch.cuda.synchronize()
    print("fp8 movers ok", flush=True)


def ring_fp8_4ranks():
    n, r = 4, 4
    q = torch.randn(1, 4, 128 * n, 128, device="cuda", dtype=torch.bfloat16)
    k, v = torch.randn_like(q), torch.randn_like(q)
    qs, ks, vs = (list(t.chunk(n, dim=2)) for t in (q, k, v))
    qs, ks, vs = ([x.contiguous() for x in t] for t in (qs, ks, vs))
    mesh = fu.make_mesh(n, r)
    for fp8 in (True, False):
        opts = fu.CommOptions(fp8_kv=fp8, pipelined_ring=True, check_finite=False)
        fu.run_protocol(n, lambda ctx: fu.usp_attention(ctx, qs[ctx.rank()], ks[ctx.rank()],
                                                        vs[ctx.rank()], mesh, opts))
    torch.cuda.synchronize()
    print("4-rank pipelined ring (fp8 + bf16) ok", flush=True)


def ulysses_fp8_u2():
    n, r = 4, 2
    q = torch.randn(1, 8, 64 * n, 128, device="cuda")
    k, v = torch.randn_like(q), torch.randn_like(q)
    qs, ks, vs = ([x.contiguous() for x in t.chunk(n, dim=2)] for t in (q, k, v))
    mesh = fu.make_mesh(n, r)
    opts = fu.CommOptions(fp8_kv=True, fp8_block=1, pipelined_ring=True, check_finite=True)
    fu.run_protocol(n, lambda ctx: fu.usp_attention_with_lse(ctx, qs[ctx.rank()], ks[ctx.rank()],
                                                             vs[ctx.rank()], mesh, opts))
    torch.cuda.synchronize()
    print("U=2 R=2 per-block FP8 f32-input layer with LSE ok", flush=True)


def fp8_pack_u4():
    # FP8 input reshard at U = 4, per-tensor scales: the one-launch cooperative amax + pack
    n = 4
    q = torch.randn(1, 8, 64 * n, 128, device="cuda", dtype=torch.bfloat16)
    k, v = torch.randn_like(q), torch.randn_like(q)
    qs, ks, vs = ([x.contiguous() for x in t.chunk(n, dim=2)] for t in (q, k, v))
    mesh = fu.make_mesh(n, 1)
    opts = fu.CommOptions(fp8_kv=True, check_finite=False)
    fu.run_protocol(n, lambda ctx: fu.usp_attention(ctx, qs[ctx.rank()], ks[ctx.rank()],
                                                    vs[ctx.rank()], mesh, opts))
    torch.cuda.synchronize()
    print("U=4 FP8 per-tensor layer (one-launch pack) ok", flush=True)


CASES = {"fp8pack": fp8_pack_u4, "attention": attention, "staging": staging, "fp8": fp8_movers, "ring": ring_fp8_4ranks,
         "usp": ulysses_fp8_u2}

if __name__ == "__main__":
    for name in sys.argv[1:] or list(CASES):
        CASES[name]()

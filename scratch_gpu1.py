# quick first-light check on the GPU (scratch; superseded by tests/)
import sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2602_10940_b200 as fu
from oracle import restate as R
torch.manual_seed(0)
dev = "cuda"
# fp8 codec
x = torch.randn(1 << 20, device=dev) * 100
x = torch.cat([x, torch.tensor([0., -0., 448, 449, 464, 465, 1000, float('inf'), -float('inf'), -1000, 2**-10, 2**-9, 3*2**-11], device=dev)])
c = fu.encode_e4m3(x).cpu().numpy(); c2 = R.encode_e4m3(x.cpu().numpy())
print("encode eq", np.array_equal(c, c2), (c != c2).sum())
xf = torch.randn(1, 24, 576, 128, device=dev) * 3
q = fu.quantize(xf); cr, sr = R.quantize(xf.cpu().numpy())
print("quantize codes eq", np.array_equal(q.codes.cpu().numpy(), cr), "scale", q.scale, float(sr), q.scale == float(sr))
# attention
for (h, sq, skv) in [(1, 128, 128), (2, 256, 256), (2, 200, 130), (3, 512, 1000), (24, 4608, 4608)]:
    qq = R.round_bf16(R.rng_tensor(42, (1, h, sq, 128)))
    kk = R.round_bf16(R.rng_tensor(43, (1, h, skv, 128)))
    vv = R.round_bf16(R.rng_tensor(44, (1, h, skv, 128)))
    tq, tk, tv = (torch.from_numpy(a).to(dev).to(torch.bfloat16) for a in (qq, kk, vv))
    res = fu.attention_with_lse(tq, tk, tv)
    torch.cuda.synchronize()
    o = res.out.cpu().numpy(); l = res.lse.cpu().numpy()
    if h * sq * skv <= 3 * 512 * 1000:
        ro, rl = R.attention_with_lse(qq, kk, vv)
    else:
        hs = slice(0, 2)
        ro, rl = R.attention_with_lse(qq[:, hs, :512], kk[:, hs], vv[:, hs]); o = o[:, hs, :512]; l = l[:, hs, :512]
    rel = np.linalg.norm(o - ro) / np.linalg.norm(ro)
    print(f"attn h={h} sq={sq} skv={skv}: relL2={rel:.3e} lse maxabs={np.abs(l - rl).max():.3e}", flush=True)
# timing FLUX
h, s = 24, 4608
tq = torch.randn(1, h, s, 128, device=dev, dtype=torch.bfloat16)
tk = torch.randn(1, h, s, 128, device=dev, dtype=torch.bfloat16)
tv = torch.randn(1, h, s, 128, device=dev, dtype=torch.float16)
for _ in range(3): fu.attention_with_lse(tq, tk, tv, out_dtype=torch.float16)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): fu.attention_with_lse(tq, tk, tv, out_dtype=torch.float16)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"FLUX attention: {ms*1000:.1f} us  {4*h*s*s*128/ms/1e9:.1f} TFLOP/s")

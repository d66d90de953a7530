"""A few USP layers on a virtual mesh (n ranks as threads on cuda:0), for ncu launch lists of
the data-movement kernels (pack / unpack / quantize / dequantize / prologue).
usage: python tools/mesh_layer_once.py N R SEQ [fp8|fp8block|bf16] [prologue]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_10940_b200 as fu

n, r, s = (int(x) for x in sys.argv[1:4])
mode = sys.argv[4] if len(sys.argv) > 4 else "bf16"
use_pro = len(sys.argv) > 5 and sys.argv[5] == "prologue"
h, d = 24, 128
sl = s // n
g = torch.Generator(device="cuda"); g.manual_seed(3)
full = [torch.empty(1, h, s, d, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1, generator=g) for _ in range(3)]
shards = [[t[:, :, i * sl:(i + 1) * sl].contiguous() for i in range(n)] for t in full]
mesh = fu.make_mesh(n, r)
opts = fu.CommOptions(fp8_kv=mode.startswith("fp8"), fp8_block=int(mode == "fp8block"),
                      pipelined_ring=True, out_dtype=torch.float16, check_finite=False)
pro = None
if use_pro:
    cos, sin = fu.rope_tables(s, d, device="cuda")
    pro = fu.QKPrologue(q_norm_weight=torch.ones(d, device="cuda"), k_norm_weight=torch.ones(d, device="cuda"),
                        rope_cos=cos, rope_sin=sin)


def prog(ctx):
    k = ctx.rank()
    for _ in range(3):
        if pro is None:
            fu.usp_attention(ctx, shards[0][k], shards[1][k], shards[2][k], mesh, opts)
        else:
            fu.usp_attention(ctx, shards[0][k], shards[1][k], shards[2][k], mesh, opts, prologue=pro)
    torch.cuda.current_stream().synchronize()


fu.run_protocol(n, prog)
# calibration: torch's own device copies of one rank's Q/K/V bytes (same ncu settings)
cal = torch.empty(3 * shards[0][0].numel(), device="cuda", dtype=torch.bfloat16)
src = torch.cat([shards[t][0].flatten() for t in range(3)])
for _ in range(3):
    cal.copy_(src)
torch.cuda.synchronize()
print("done")

"""GPU parity at the BASELINE configurations' own shapes (BASELINE.json configs[2..4]), with
every rank of the mesh as a thread on one B200 (in-process fabric), checked on head / row
subsets against the oracle (full-sequence attention for those rows in float64, and for the FP8
configuration the reference quantizer's own per-rank K/V: oracle/_ref = fp8.cpp:107-130).

  cfg3  S=16896 (2048x2048 image + 512 text), H=24, U=2 R=4 on 8 ranks: serial and pipelined
        ring (protocols.cpp:237-319), pipelined bit-identical to serial;
  cfg4  FLUX S=4608 H=24, U=8: FP8 K/V per-tensor and per-block against the reference
        quantizer's dequantized K/V (protocols.cpp:139-179), plus the BF16 wire;
  cfg5  Qwen-Image-shaped S=7168 H=24, U=4 R=2 on 8 ranks, three layers back to back (eager:
        the in-process fabric is not graph-capturable; CUDA-graph replay of the same 3-layer
        stack is checked bit-identical to eager at world 1 below)."""
import numpy as np
import pytest
import torch

from oracle import ref, ref_available
from oracle import restate as R

pytestmark = pytest.mark.gpu

REL = 1e-3


def rel_l2(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def tensors(shape, seed):
    g = torch.Generator().manual_seed(seed)
    return [torch.empty(shape).uniform_(-1, 1, generator=g).bfloat16() for _ in range(3)]


def run(fu, q, k, v, n, r, **opt):
    shard = [[x.contiguous().cuda() for x in t.chunk(n, dim=2)] for t in (q, k, v)]
    mesh = fu.make_mesh(n, r)
    opts = fu.CommOptions(check_finite=False, out_dtype=torch.float32, **opt)
    rep = fu.run_protocol(n, lambda ctx: fu.usp_attention(
        ctx, shard[0][ctx.rank()], shard[1][ctx.rank()], shard[2][ctx.rank()], mesh, opts))
    return torch.cat(rep.results, dim=2)


def subset_ref(q, k, v, heads, rows):
    o, _ = R.attention_with_lse(q[:, heads][:, :, rows].float().numpy(), k[:, heads].float().numpy(),
                                v[:, heads].float().numpy())
    return o


def test_cfg3_ring_heavy_s16896(cuda, fu):
    s, h = 16896, 24
    q, k, v = tensors((1, h, s, 128), 3)
    rows = np.r_[0:64, 8448:8512, s - 64:s]
    heads = [0, 13, 23]
    want = subset_ref(q, k, v, heads, rows)
    outs = {}
    for pipelined in (False, True):
        got = run(fu, q, k, v, 8, 4, pipelined_ring=pipelined)
        outs[pipelined] = got
        assert rel_l2(got[:, heads][:, :, rows].cpu().numpy(), want) <= REL
    assert torch.equal(outs[False], outs[True])


def fp8_kv_reference(x, n, per_block):
    """Each rank quantizes its whole local shard (fp8.cpp:107-123; per-block: per (b,h) slab)
    with the reference's own quantizer; the receivers hold decode(code) * scale."""
    parts = []
    for sh in x.chunk(n, dim=2):
        a = sh.float().numpy()
        if not per_block:
            c, sc = ref.quantize(a)
            parts.append(ref.dequantize(c, sc))
        else:
            d = np.empty_like(a)
            for hh in range(a.shape[1]):
                c, sc = ref.quantize(a[:, hh:hh + 1])
                d[:, hh:hh + 1] = ref.dequantize(c, sc)
            parts.append(d)
    return torch.from_numpy(np.concatenate(parts, axis=2))


@pytest.mark.parametrize("mode", ["bf16", "fp8", "fp8_block"])
def test_cfg4_flux_u8(cuda, fu, mode):
    if mode != "bf16" and not ref_available():
        pytest.skip("oracle/_ref not built")
    s, h = 4608, 24
    q, k, v = tensors((1, h, s, 128), 4)
    k[:, 5] *= 9  # heads of different range: per-block scales differ from the per-tensor one
    v[:, 17] *= 0.05
    rows = np.r_[0:64, 2304:2368, s - 64:s]
    heads = [0, 5, 17, 23]
    if mode == "bf16":
        got = run(fu, q, k, v, 8, 1)
        assert rel_l2(got[:, heads][:, :, rows].cpu().numpy(), subset_ref(q, k, v, heads, rows)) <= REL
        return
    pb = mode == "fp8_block"
    kd, vd = fp8_kv_reference(k, 8, pb), fp8_kv_reference(v, 8, pb)
    want = subset_ref(q, kd, vd, heads, rows)
    got = run(fu, q, k, v, 8, 1, fp8_kv=True, fp8_block=int(pb))
    # same FP8 values as the reference; what remains is the bf16/f16 tensor-core arithmetic
    assert rel_l2(got[:, heads][:, :, rows].cpu().numpy(), want) <= 2e-3


def test_cfg5_qwen_three_layers(cuda, fu):
    s, h, layers = 7168, 24, 3
    rows = np.r_[0:64, 3584:3648, s - 64:s]
    heads = [0, 11, 23]
    n, r = 8, 2
    per_layer = [tensors((1, h, s, 128), 50 + i) for i in range(layers)]
    shards = [[[x.contiguous().cuda() for x in t.chunk(n, dim=2)] for t in lay] for lay in per_layer]
    mesh = fu.make_mesh(n, r)
    opts = fu.CommOptions(check_finite=False, out_dtype=torch.float32, pipelined_ring=True)
    rep = fu.run_protocol(n, lambda ctx: [fu.usp_attention(
        ctx, sh[0][ctx.rank()], sh[1][ctx.rank()], sh[2][ctx.rank()], mesh, opts) for sh in shards])
    for i, (q, k, v) in enumerate(per_layer):
        got = torch.cat([res[i] for res in rep.results], dim=2)
        assert rel_l2(got[:, heads][:, :, rows].cpu().numpy(), subset_ref(q, k, v, heads, rows)) <= REL


def test_cfg5_graph_replay_matches_eager_world1(cuda, fu):
    # the 3-layer stack of Qwen-shaped layers under one CUDA graph vs eager, bit for bit
    L, s, h = 3, 7168, 24
    q = torch.randn(L, 1, h, s // 8, 128, device="cuda", dtype=torch.bfloat16)
    k, v = torch.randn_like(q), torch.randn_like(q)
    out = torch.empty(L, 1, h, s // 8, 128, device="cuda", dtype=torch.float16)
    mesh = fu.make_mesh(1, 1)
    opts = fu.CommOptions(out_dtype=torch.float16, check_finite=False)

    def prog(ctx):
        eager = [fu.usp_attention(ctx, q[i], k[i], v[i], mesh, opts) for i in range(L)]
        g = fu.LayerGraph(ctx, q, k, v, out, mesh, opts, layers=L)
        g.launch()
        torch.cuda.current_stream().synchronize()
        g.close()
        return eager

    eager = fu.run_protocol(1, prog).results[0]
    for i in range(L):
        assert torch.equal(out[i], eager[i])


def test_graph_survives_eager_workspace_growth(cuda, fu):
    # a captured graph owns its workspace; a later eager call that needs a
    # bigger arena on the same context must not free memory the graph replays
    small = torch.randn(1, 1, 8, 512, 128, device="cuda", dtype=torch.bfloat16)
    out = torch.empty(1, 1, 8, 512, 128, device="cuda", dtype=torch.float16)
    big = torch.randn(1, 24, 4608, 128, device="cuda", dtype=torch.bfloat16)
    mesh = fu.make_mesh(1, 1)
    opts = fu.CommOptions(out_dtype=torch.float16, check_finite=False)

    def prog(ctx):
        want = fu.usp_attention(ctx, small[0], small[0], small[0], mesh, opts)
        g = fu.LayerGraph(ctx, small, small, small, out, mesh, opts, layers=1)
        fu.usp_attention(ctx, big, big, big, mesh, opts)  # regrows the context's arena
        out.zero_()
        g.launch()
        torch.cuda.current_stream().synchronize()
        ok = torch.equal(out[0], want)
        with pytest.raises(fu.FuspError, match="live graph"):
            fu._lib.check(fu._lib.lib().fusp_ctx_destroy(ctx.handle))
        g.close()
        return ok

    assert fu.run_protocol(1, prog).results[0]

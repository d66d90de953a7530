"""GPU parity on inputs the reference accepts but bf16 / f16 staging would mangle.

The reference computes in f32 on whatever finite values it is given (tensor.cpp:143-181,
protocols.cpp:97-105).  fastusp stages operands into the tensor cores' 16-bit types:
  * f32 Q, K run the f16 MMA (11 significant bits, not bf16's 8);
  * every staging into f16 from a wider range (f32, bf16, FP8 decode * scale) is range-guarded
    per head by an exact power of two that the kernel folds back (fastusp_internal.h).
These tests feed genuine f32 data (NOT bf16-representable) and magnitudes far outside f16's
range (|V| ~ 1e5 overflows f16, |V| ~ 1e-6 is f16-subnormal) through the C ABI, and compare
with the reference library itself (oracle/_ref, uspsim compiled from the reference sources).

Bars (stated here, cited by INTEGRATION.md): output rel-L2 <= 1e-3 against the reference's
f32 result; natural-log LSE |delta| <= 5e-3 for f32 inputs (f16 Q.K^T: ~2^-11 relative logit
error; bf16-exact inputs keep the 1e-4 bar of test_gpu_kernels.py); FP8 path against the
reference's own FP8 output <= 2e-3."""
import numpy as np
import pytest
import torch

from oracle import ref, ref_available
from oracle import restate as R

pytestmark = pytest.mark.gpu

REL_L2 = 1e-3
REL_L2_FP8 = 2e-3
LSE_F32 = 5e-3


@pytest.fixture(scope="module", autouse=True)
def _need_ref():
    if not ref_available():
        pytest.skip("oracle/_ref not built")


def rel_l2(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def f32_qkv(shape, lo, hi, seeds=(71, 72, 73)):
    """Genuine f32 values (the reference RNG stream, never rounded to bf16)."""
    q, k, v = (R.rng_tensor(s, shape, lo, hi).astype(np.float32) for s in seeds)
    assert not np.array_equal(q, R.round_bf16(q))  # really not bf16-representable
    return q, k, v


def gpu(x, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda().to(dtype)


def run_usp(fu, q, k, v, n, r, dtype=torch.float32, **opt):
    qs, ks, vs = ([gpu(s, dtype) for s in R.split_sequence(t, n)] for t in (q, k, v))
    mesh = fu.make_mesh(n, r)
    opts = fu.CommOptions(**opt)
    rep = fu.run_protocol(n, lambda ctx: fu.usp_attention(
        ctx, qs[ctx.rank()], ks[ctx.rank()], vs[ctx.rank()], mesh, opts))
    return torch.cat([o.float() for o in rep.results], dim=2).cpu().numpy(), rep


@pytest.mark.parametrize("lo,hi", [(-1.0, 1.0), (-3.0, 3.0)])
def test_attention_with_lse_f32_inputs(cuda, fu, lo, hi):
    q, k, v = f32_qkv((1, 4, 640, 128), lo, hi)
    want_o, want_l = ref.attention_with_lse(q, k, v)
    res = fu.attention_with_lse(gpu(q), gpu(k), gpu(v))
    got_o, got_l = res.out.cpu().numpy(), res.lse.cpu().numpy()
    assert rel_l2(got_o, want_o) <= REL_L2
    assert np.abs(got_l - want_l).max() <= LSE_F32


@pytest.mark.parametrize("lo,hi", [(-1.0, 1.0), (-3.0, 3.0)])
@pytest.mark.parametrize("pipelined", [False, True])
def test_usp_f32_inputs_u2_r2(cuda, fu, lo, hi, pipelined):
    h, s = 8, 256
    q, k, v = f32_qkv((1, h, s, 128), lo, hi)
    want = ref.usp_attention(q, k, v, 4, 2, pipelined=pipelined)
    got, rep = run_usp(fu, q, k, v, 4, 2, pipelined_ring=pipelined)
    assert rel_l2(got, want) <= REL_L2
    # f32 inputs keep the reference's f32 wire: SPEC.md:349 closed forms at w = 4, exactly
    _, a2a, snd = ref.usp_attention(q, k, v, 4, 2, traffic=True)
    assert [t[0] for t in rep.traffic] == [int(x) for x in a2a]
    assert [t[1] for t in rep.traffic] == [int(x) for x in snd]


@pytest.mark.parametrize("lo,hi", [(-1.0, 1.0), (-3.0, 3.0)])
def test_ring_f32_inputs(cuda, fu, lo, hi):
    q, k, v = f32_qkv((1, 4, 256, 128), lo, hi)
    want_o, want_l = ref.ring_attention(q, k, v, 4, pipelined=True)
    qs, ks, vs = ([gpu(x) for x in R.split_sequence(t, 4)] for t in (q, k, v))
    rep = fu.run_protocol(4, lambda ctx: fu.ring_attention_pipelined(
        ctx, qs[ctx.rank()], ks[ctx.rank()], vs[ctx.rank()]))
    out = torch.cat([x.out for x in rep.results], dim=2).cpu().numpy()
    lse = torch.cat([x.lse for x in rep.results], dim=2).cpu().numpy()
    assert rel_l2(out, want_o) <= REL_L2
    assert np.abs(lse - want_l).max() <= LSE_F32


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("vscale", [1e5, 1e-6])
def test_v_range_guard_attention(cuda, fu, dtype, vscale):
    q, k, v = f32_qkv((1, 3, 384, 128), -1.0, 1.0)
    v = (v * vscale).astype(np.float32)
    v[:, 1] /= vscale  # one head in range: only the out-of-range heads take the guarded path
    if dtype == torch.bfloat16:
        q, k, v = R.round_bf16(q), R.round_bf16(k), R.round_bf16(v)
    want_o, want_l = ref.attention_with_lse(q, k, v)
    res = fu.attention_with_lse(gpu(q, dtype), gpu(k, dtype), gpu(v, dtype))
    got = res.out.cpu().numpy()
    assert np.isfinite(got).all()
    for h in range(3):  # per head: the in-range head must not be disturbed by the others
        assert rel_l2(got[:, h], want_o[:, h]) <= REL_L2
    bar = 1e-4 if dtype == torch.bfloat16 else LSE_F32
    assert np.abs(res.lse.cpu().numpy() - want_l).max() <= bar


@pytest.mark.parametrize("qk", [(1e5, 1e-5), (1e-4, 1e4)])
def test_qk_range_guard_f32(cuda, fu, qk):
    # Q beyond f16's range and K in its subnormals (or the reverse); the logits stay O(1)
    q, k, v = f32_qkv((1, 2, 256, 128), -1.0, 1.0)
    q, k = (q * qk[0]).astype(np.float32), (k * qk[1]).astype(np.float32)
    want_o, want_l = ref.attention_with_lse(q, k, v)
    res = fu.attention_with_lse(gpu(q), gpu(k), gpu(v))
    assert rel_l2(res.out.cpu().numpy(), want_o) <= REL_L2
    assert np.abs(res.lse.cpu().numpy() - want_l).max() <= LSE_F32


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("vscale", [1e5, 1e-6])
@pytest.mark.parametrize("pipelined", [False, True])
def test_v_range_guard_usp(cuda, fu, dtype, vscale, pipelined):
    q, k, v = f32_qkv((1, 8, 256, 128), -1.0, 1.0)
    v = (v * vscale).astype(np.float32)
    if dtype == torch.bfloat16:
        q, k, v = R.round_bf16(q), R.round_bf16(k), R.round_bf16(v)
    want = ref.usp_attention(q, k, v, 4, 2)
    got, _ = run_usp(fu, q, k, v, 4, 2, dtype=dtype, pipelined_ring=pipelined)
    assert np.isfinite(got).all()
    assert rel_l2(got, want) <= REL_L2


@pytest.mark.parametrize("vscale", [1e5, 1e-6])
def test_range_guard_fp8_path(cuda, fu, vscale):
    # FP8 K/V decode to decode(code) * scale, whose range follows the data: staged guarded
    q, k, v = f32_qkv((1, 8, 256, 128), -1.0, 1.0)
    q = R.round_bf16(q * 1e5)          # Q is staged bf16 -> f16 on the FP8 path
    k = R.round_bf16(k * 1e-5)
    v = R.round_bf16(v * vscale)
    want = ref.usp_attention(q, k, v, 4, 2, fp8=True)
    got, _ = run_usp(fu, q, k, v, 4, 2, dtype=torch.bfloat16, fp8_kv=True)
    assert np.isfinite(got).all()
    assert rel_l2(got, want) <= REL_L2_FP8


def test_range_guard_u1_and_ulysses(cuda, fu):
    # U = 1 staging (no wire) and the Ulysses-only unpack, f32 |V| ~ 1e5
    q, k, v = f32_qkv((1, 4, 256, 128), -1.0, 1.0)
    v = (v * 1e5).astype(np.float32)
    want = ref.usp_attention(q, k, v, 1, 1)
    got, _ = run_usp(fu, q, k, v, 1, 1)
    assert rel_l2(got, want) <= REL_L2
    want = ref.usp_attention(q, k, v, 4, 1)
    got, _ = run_usp(fu, q, k, v, 4, 1)
    assert rel_l2(got, want) <= REL_L2


@pytest.mark.parametrize("b,h,n,r", [(2, 6, 2, 1), (1, 24, 1, 1), (1, 12, 4, 2)])
def test_host_path_uneven_chunks(cuda, fu, b, h, n, r):
    # fusp_usp_attention_host pipelines head chunks of halving size ([12, 6, 3, 2, 1] at H=24):
    # every chunk is a valid layer, the result is the unchunked one
    q, k, v = f32_qkv((b, h, 64 * n, 128), -1.0, 1.0)
    want = ref.usp_attention(q, k, v, n, r)
    qs, ks, vs = ([torch.from_numpy(np.ascontiguousarray(s)) for s in R.split_sequence(t, n)]
                  for t in (q, k, v))
    mesh = fu.make_mesh(n, r)
    rep = fu.run_protocol(n, lambda ctx: fu.usp_attention_host(ctx, qs[ctx.rank()], ks[ctx.rank()],
                                                               vs[ctx.rank()], mesh))
    got = torch.cat(rep.results, dim=2).numpy()
    assert rel_l2(got, want) <= REL_L2


@pytest.mark.parametrize("fp8", [False, True])
def test_ragged_batch2_guarded(cuda, fu, fp8):
    # S/N = 100 (not a multiple of the 128-row tile), B = 2, f32 inputs, one loud V head
    n, r = 4, 2
    q, k, v = f32_qkv((2, 8, 100 * n, 128), -1.0, 1.0)
    v[:, 3] *= 1e5
    if fp8:
        q, k, v = R.round_bf16(q), R.round_bf16(k), R.round_bf16(v)
        want = ref.usp_attention(q, k, v, n, r, fp8=True)
        got, _ = run_usp(fu, q, k, v, n, r, dtype=torch.bfloat16, fp8_kv=True, pipelined_ring=True)
        assert rel_l2(got, want) <= REL_L2_FP8
    else:
        want = ref.usp_attention(q, k, v, n, r)
        got, _ = run_usp(fu, q, k, v, n, r, pipelined_ring=True)
        assert rel_l2(got, want) <= REL_L2
    assert np.isfinite(got).all()


def test_graph_replay_guarded_f32(cuda, fu):
    # the range guard's exponents are device state: a captured layer replays them correctly
    L = 2
    x = [torch.from_numpy(t).cuda() for t in f32_qkv((1, 4, 512, 128), -1.0, 1.0)]
    q, k, v = (torch.stack([t, t * 3]) for t in x)
    v[1] *= 1e5
    out = torch.empty(L, 1, 4, 512, 128, device="cuda", dtype=torch.float32)
    mesh = fu.make_mesh(1, 1)
    opts = fu.CommOptions(out_dtype=torch.float32, check_finite=False)

    def prog(ctx):
        eager = [fu.usp_attention(ctx, q[i], k[i], v[i], mesh, opts) for i in range(L)]
        g = fu.LayerGraph(ctx, q, k, v, out, mesh, opts, layers=L)
        for _ in range(2):
            g.launch()
        torch.cuda.current_stream().synchronize()
        g.close()
        return eager

    eager = fu.run_protocol(1, prog).results[0]
    for i in range(L):
        assert torch.equal(out[i], eager[i])
        want, _ = ref.attention_with_lse(q[i].cpu().numpy(), k[i].cpu().numpy(), v[i].cpu().numpy())
        assert rel_l2(out[i].cpu().numpy(), want) <= REL_L2


def test_stage_f16_exact_power_of_two(cuda, fu):
    # fusp_stage_f16: y * 2^exps == x wherever x is an f16 value times a power of two
    x = torch.randn(5, 256, 128, device="cuda").half().float()
    scale = torch.tensor([1.0, 2.0 ** 30, 2.0 ** -30, 1e-3, 2.0 ** 20], device="cuda")
    xs = x * scale[:, None, None]
    y, e = fu.stage_f16(xs)
    back = y.float() * torch.pow(2.0, e.float())[:, None, None]
    assert torch.equal(back[[0, 1, 2, 4]], xs[[0, 1, 2, 4]])
    # max|x| ~ 4: in range; 2^30 / 2^20 above 2^15; 2^-30 and 1e-3 (max ~4e-3) below 2^-6
    assert e[0].item() == 0 and e[1].item() > 0 and e[2].item() < 0 and e[3].item() < 0 and e[4].item() > 0
    assert torch.isfinite(y.float()).all()

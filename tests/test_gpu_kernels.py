"""GPU parity of the single-GPU kernels against the oracle (tensor.cpp / fp8.cpp).

Bars: byte/integer work bit-exact; attention rel-L2 <= 1e-3 on O against the fp32
reference (north star) and |dLSE| <= 1e-4; merge within 1e-6 (fp32 elementwise)."""
import hashlib
import math

import numpy as np
import pytest
import torch

from oracle import restate as R
from oracle.make_golden import ATTN_CASES, fp8_grid, qkv

pytestmark = pytest.mark.gpu

GOLD = __import__("os").path.join(__import__("os").path.dirname(__file__), "golden")
REL_L2 = 1e-3
LSE_TOL = 1e-4


def gold(name):
    return np.load(f"{GOLD}/{name}.npz")


def rel_l2(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def T(x, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda().to(dtype)


# ---- E4M3 codec -----------------------------------------------------------------------------------
def test_encode_bit_exact_golden(cuda, fu):
    x = fp8_grid()
    got = fu.encode_e4m3(T(x)).cpu().numpy()
    assert np.array_equal(got, gold("fp8")["enc_codes"])


def test_encode_bit_exact_random_and_nan(cuda, fu):
    rs = np.random.RandomState(3)
    x = np.concatenate([rs.standard_normal(1 << 20).astype(np.float32) * s for s in (1e-3, 1, 300)])
    bits = np.array([0x7FC00000, 0xFFC00000, 0x7F800001, 0xFF800001], np.uint32).view(np.float32)
    x = np.concatenate([x, bits])
    assert np.array_equal(fu.encode_e4m3(T(x)).cpu().numpy(), R.encode_e4m3(x))


def test_decode_all_codes(cuda, fu):
    c = np.arange(256, dtype=np.uint8)
    got = fu.decode_e4m3(T(c, torch.uint8)).cpu().numpy()
    assert np.array_equal(got, gold("fp8")["dec_vals"], equal_nan=True)
    assert math.copysign(1.0, got[0x80]) < 0


@pytest.mark.parametrize("name,shape,lo,hi,seed", [
    ("u1", (1, 4, 16, 128), -1, 1, 11), ("u3", (2, 3, 40, 128), -3, 3, 12)])
def test_quantize_bit_exact_golden(cuda, fu, name, shape, lo, hi, seed):
    g = gold("fp8")
    t = R.rng_tensor(seed, shape, lo, hi)
    q = fu.quantize(T(t))
    assert np.array_equal(q.codes.cpu().numpy(), g[f"q_{name}_codes"])
    assert q.scale == float(g[f"q_{name}_scale"][0])


def test_quantize_flux_shape_bit_exact(cuda, fu):
    # the FLUX U=8 local K [1,24,576,128] (SURVEY 7.2 minimum slice), bf16 input
    g = gold("fp8")
    t = R.round_bf16(R.rng_tensor(43, (1, 24, 576, 128)))
    for dt in (torch.float32, torch.bfloat16):
        q = fu.quantize(T(t, dt))
        digest = hashlib.sha256(q.codes.cpu().numpy().tobytes()).digest()
        assert digest == g["q_flux_u8_k_sha256"].tobytes()
        assert q.scale == float(g["q_flux_u8_k_scale"][0])


def test_quantize_spec_examples(cuda, fu):
    q = fu.quantize(T(np.array([448, -224, 0], np.float32).reshape(1, 1, 1, 3)))
    assert q.codes.cpu().numpy().ravel().tolist() == [0x7E, 0xF6, 0x00] and q.scale == 1.0
    q = fu.quantize(torch.zeros(1, 2, 3, 4, device="cuda"))
    assert q.scale == 1.0 and int(q.codes.sum()) == 0
    deq = fu.dequantize(fu.quantize(T(np.array([448, -224, 0], np.float32).reshape(1, 1, 1, 3))))
    assert deq.cpu().numpy().ravel().tolist() == [448.0, -224.0, 0.0]


@pytest.mark.parametrize("scale", [1e-6, 1.0, 1e4])
def test_quantize_dequantize_match_restatement(cuda, fu, scale):
    t = (np.random.RandomState(5).standard_normal((1, 8, 100, 128)) * scale).astype(np.float32)
    q = fu.quantize(T(t))
    c, s = R.quantize(t)
    assert np.array_equal(q.codes.cpu().numpy(), c) and q.scale == float(s)
    assert np.array_equal(fu.dequantize(q).cpu().numpy(), R.dequantize(c, s))


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_quantize_blocks_equal_reference_per_slice(cuda, fu, dtype):
    # per-block = uspsim::quantize applied to every (b,h) slab on its own (bit-exact)
    t = R.rng_tensor(77, (2, 5, 96, 128), -3, 3)
    t[1, 2] *= 50.0  # one slab with a very different range
    t = R.round_bf16(t)  # the bf16 run must see exactly the oracle's values
    codes, scales = fu.quantize_blocks(T(t, dtype), 96 * 128)
    codes, scales = codes.cpu().numpy(), scales.cpu().numpy()
    for b in range(2):
        for h in range(5):
            c, s = R.quantize(t[b:b + 1, h:h + 1])
            assert np.array_equal(codes[b:b + 1, h:h + 1], c) and scales[b * 5 + h] == s
    back = fu.dequantize_blocks(T(codes, torch.uint8), T(scales), 96 * 128).cpu().numpy()
    assert np.array_equal(back, R.fake_quant(t, per_block=True))


def test_quantize_words_reset_between_calls(cuda, fu):
    # the amax pass finalizes the scales in its last CTA and leaves its zero words zero: a large
    # amax followed by a small one (and block counts that change) must each be bit-exact, and
    # so must the ring-hop requantize of the multi-scale codes just produced
    for i, (lo, hi, block) in enumerate([(-300, 300, 64 * 128), (-0.01, 0.01, 64 * 128),
                                         (-5, 5, 4 * 64 * 128), (-1e-3, 1e-3, 2 * 64 * 128)]):
        t = R.round_bf16(R.rng_tensor(500 + i, (1, 4, 64, 128), lo, hi))
        nb = t.size // block
        flat = t.reshape(nb, block)
        for _ in range(2):
            codes, scales = fu.quantize_blocks(T(t, torch.bfloat16), block)
            codes, scales = codes.cpu().numpy().reshape(nb, block), scales.cpu().numpy()
            for j in range(nb):
                c, sc = R.quantize(flat[j:j + 1])
                assert np.array_equal(codes[j], c.reshape(-1)) and scales[j] == sc
        deq = np.concatenate([R.dequantize(codes[j], scales[j]) for j in range(nb)])
        wc, ws = R.quantize(deq)
        for _ in range(2):
            q2 = fu.requantize(T(codes.reshape(-1), torch.uint8), T(scales[:nb]), block)
            assert np.array_equal(q2.codes.cpu().numpy().reshape(-1), wc.reshape(-1))
            assert q2.scale == ws


def test_quantize_rejects_non_finite_like_reference(cuda, fu):
    t = torch.zeros(1, 1, 2, 8, device="cuda")
    t[0, 0, 1, 3] = float("inf")
    with pytest.raises(fu.InvalidArgument, match="non-finite element at flat index 11"):
        fu.quantize(t)


# ---- attention_with_lse ---------------------------------------------------------------------------
@pytest.mark.parametrize("name,b,h,sq,skv", ATTN_CASES)
def test_attention_vs_reference_golden(cuda, fu, name, b, h, sq, skv):
    g = gold("attention")
    q, k, v = qkv((b, h, sq, 128), (b, h, skv, 128))
    r = fu.attention_with_lse(T(q, torch.bfloat16), T(k, torch.bfloat16), T(v, torch.bfloat16))
    assert rel_l2(r.out.cpu().numpy(), g[f"{name}_out"]) <= REL_L2
    assert np.abs(r.lse.cpu().numpy() - g[f"{name}_lse"]).max() <= LSE_TOL


@pytest.mark.parametrize("in_dtype", [torch.float32, torch.bfloat16, torch.float16])
@pytest.mark.parametrize("out_dtype", [torch.float32, torch.float16])
def test_attention_dtypes(cuda, fu, in_dtype, out_dtype):
    q, k, v = qkv((1, 3, 300, 128), (1, 3, 517, 128))
    ro, rl = R.attention_with_lse(q, k, v)
    r = fu.attention_with_lse(T(q, in_dtype), T(k, in_dtype), T(v, in_dtype), out_dtype=out_dtype)
    assert rel_l2(r.out.float().cpu().numpy(), ro) <= REL_L2
    assert np.abs(r.lse.cpu().numpy() - rl).max() <= LSE_TOL


def test_attention_bf16_output_documented_bound(cuda, fu):
    # bf16 output alone costs ~1.65e-3; allowed but bounded
    q, k, v = qkv((1, 2, 256, 128), (1, 2, 256, 128))
    ro, _ = R.attention_with_lse(q, k, v)
    r = fu.attention_with_lse(T(q, torch.bfloat16), T(k, torch.bfloat16), T(v, torch.bfloat16),
                              out_dtype=torch.bfloat16)
    assert rel_l2(r.out.float().cpu().numpy(), ro) <= 3e-3


def test_attention_empty_keys_is_merge_identity(cuda, fu):
    q = torch.randn(1, 2, 7, 128, device="cuda")
    k = torch.zeros(1, 2, 0, 128, device="cuda")
    r = fu.attention_with_lse(q, k, k)
    assert torch.all(r.out == 0) and torch.all(torch.isneginf(r.lse))


def test_attention_scaled_inputs_wide_range(cuda, fu):
    # [-3, 3] inputs (SPEC.md:67 property range) stress the lazy-rescale path
    q, k, v = qkv((1, 2, 256, 128), (1, 2, 640, 128), lo=-3, hi=3)
    ro, rl = R.attention_with_lse(q, k, v)
    r = fu.attention_with_lse(T(q, torch.bfloat16), T(k, torch.bfloat16), T(v, torch.bfloat16))
    assert rel_l2(r.out.cpu().numpy(), ro) <= REL_L2
    assert np.abs(r.lse.cpu().numpy() - rl).max() <= LSE_TOL


def test_attention_increasing_max_forces_rescale(cuda, fu):
    # keys whose logits grow along the sequence: every KV tile raises the row max
    rs = np.random.RandomState(9)
    q = np.ones((1, 1, 128, 128), np.float32) * 0.5
    k = (np.linspace(0, 4, 1024)[None, None, :, None] * np.ones((1, 1, 1, 128))).astype(np.float32)
    k = R.round_bf16(k)
    v = R.round_bf16(rs.uniform(-1, 1, (1, 1, 1024, 128)).astype(np.float32))
    ro, rl = R.attention_with_lse(q, k, v)
    r = fu.attention_with_lse(T(q, torch.bfloat16), T(k, torch.bfloat16), T(v, torch.bfloat16))
    assert rel_l2(r.out.cpu().numpy(), ro) <= REL_L2
    assert np.abs(r.lse.cpu().numpy() - rl).max() <= LSE_TOL


def test_attention_convexity_and_uniform(cuda, fu):
    # outputs are convex combinations of V rows; identical keys -> mean of V
    v = torch.randn(1, 2, 300, 128, device="cuda", dtype=torch.float16)
    q = torch.randn(1, 2, 100, 128, device="cuda", dtype=torch.float16)
    k = torch.randn(1, 2, 300, 128, device="cuda", dtype=torch.float16)
    out = fu.attention_with_lse(q, k, v).out
    lo = v.float().amin(dim=2, keepdim=True) - 1e-3
    hi = v.float().amax(dim=2, keepdim=True) + 1e-3
    assert bool(((out >= lo) & (out <= hi)).all())
    ku = torch.ones_like(k)
    out = fu.attention_with_lse(q, ku, v).out
    assert torch.allclose(out, v.float().mean(dim=2, keepdim=True).expand_as(out), atol=2e-3)


def test_attention_flux_full_size(cuda, fu):
    # FLUX layer [1,24,4608,128] on one GPU: head subset vs the oracle, plus the
    # size-independent chunk-equivalence property over the whole tensor.
    h, s = 24, 4608
    q, k, v = qkv((1, h, s, 128), (1, h, s, 128))
    tq, tk, tv = (T(x, torch.bfloat16) for x in (q, k, v))
    r = fu.attention_with_lse(tq, tk, tv)
    rows = slice(0, 384)
    ro, rl = R.attention_with_lse(q[:, :2, rows], k[:, :2], v[:, :2])
    assert rel_l2(r.out[:, :2, rows].cpu().numpy(), ro) <= REL_L2
    assert np.abs(r.lse[:, :2, rows].cpu().numpy() - rl).max() <= LSE_TOL
    a = fu.attention_with_lse(tq, tk[:, :, :2000], tv[:, :, :2000])
    b = fu.attention_with_lse(tq, tk[:, :, 2000:], tv[:, :, 2000:])
    m = fu.merge_lse(a, b)
    assert rel_l2(m.out.cpu().numpy(), r.out.cpu().numpy()) <= REL_L2
    assert float((m.lse - r.lse).abs().max()) <= LSE_TOL


# ---- merge_lse ------------------------------------------------------------------------------------
def test_merge_vs_reference_golden(cuda, fu):
    g = gold("attention")
    a = fu.AttnResult(T(g["merge_o1"]), T(g["merge_l1"]))
    b = fu.AttnResult(T(g["merge_o2"]), T(g["merge_l2"]))
    m = fu.merge_lse(a, b)
    assert np.abs(m.out.cpu().numpy() - g["merge_out"]).max() <= 1e-6
    assert np.abs(m.lse.cpu().numpy() - g["merge_lse"]).max() <= 1e-6


def test_merge_identity_bit_exact(cuda, fu):
    g = gold("attention")
    a = fu.AttnResult(T(g["merge_o1"]), T(g["merge_l1"]))
    ident = fu.AttnResult.identity(a.out.shape)
    for x, y in ((a, ident), (ident, a)):
        m = fu.merge_lse(x, y)
        assert torch.equal(m.out, a.out) and torch.equal(m.lse, a.lse)


def test_merge_shape_errors(cuda, fu):
    a = fu.AttnResult.identity((1, 1, 4, 128))
    b = fu.AttnResult.identity((1, 1, 5, 128))
    with pytest.raises(fu.ShapeError, match="merge_lse: output shapes differ"):
        fu.merge_lse(a, b)


def test_attention_shape_errors(cuda, fu):
    q = torch.zeros(1, 2, 4, 128, device="cuda")
    with pytest.raises(fu.ShapeError, match="head axis mismatch"):
        fu.attention_with_lse(q, torch.zeros(1, 3, 4, 128, device="cuda"), q)
    # head dims other than 128 run on the generic kernel; D must be a multiple of 8, <= 256
    with pytest.raises(fu.ShapeError, match="D=60 unsupported"):
        x = torch.zeros(1, 1, 4, 60, device="cuda")
        fu.attention_with_lse(x, x, x)


def test_kernels_counted(cuda, fu):
    n0 = fu.kernel_launch_count()
    q = torch.randn(1, 1, 128, 128, device="cuda", dtype=torch.bfloat16)
    fu.attention_with_lse(q, q, q.half())
    torch.cuda.synchronize()
    assert fu.kernel_launch_count() > n0


def test_quantize_near_rounding_boundaries_bit_exact(cuda, fu):
    # x / scale landing within a few f32 ulps of every E4M3 rounding midpoint (normal and
    # subnormal range, both signs): the vectorised quantizer must still encode exactly like
    # the reference's IEEE division (fp8.cpp:121) -- its fast x * (1/scale) path has to defer
    # to the exact division at every one of these.
    mags = R.decode_e4m3(np.arange(0, 127, dtype=np.uint8))
    mids = (np.float32(0.5) * (mags[:-1] + mags[1:])).astype(np.float32)
    amax = np.float32(3.7)
    scale = np.float32(amax / np.float32(448.0))
    qs = []
    for m in mids:
        q = np.float32(m)
        for _ in range(8):
            q = np.nextafter(q, np.float32(0))
        for _ in range(17):
            qs.append(q)
            q = np.nextafter(q, np.float32(np.inf))
    q = np.array(qs, np.float32)
    x = (q * scale).astype(np.float32)
    x = np.concatenate([x, -x, np.array([amax], np.float32)])
    x = np.concatenate([x, np.zeros((-x.size) % 128, np.float32)])
    want, s = R.quantize(x)
    codes, scales = fu.quantize_blocks(T(x), x.size)
    assert scales.cpu().numpy()[0] == s
    got = codes.cpu().numpy()
    bad = np.flatnonzero(got != want)
    assert bad.size == 0, (bad[:5], x[bad[:5]], got[bad[:5]], want[bad[:5]])


@pytest.mark.parametrize("seg_scales", [
    [0.01, 0.01, 0.01, 0.01],          # uniform: a later ring hop, every vector copied
    [0.01, 0.0371, 0.002, 0.0371],     # the resharded first hop: senders' scales differ
    [1.0, 1.0],                        # an all-zero chunk re-quantizes to scale 1
    [3.3e-3, 1.7e-5, 2.9, 0.125, 0.125, 7.0e-2],
])
def test_requantize_ring_hop_bit_exact(cuda, fu, seg_scales):
    # quantize(dequantize(chunk)) of the ring forward (protocols.cpp:113-115, 309-310) on a
    # chunk whose segments carry different scales: codes and scale bit-exact vs the oracle,
    # including the copy path taken when a segment's scale equals the new one.
    rng = np.random.default_rng(len(seg_scales))
    seg = 1024
    codes = rng.integers(0, 256, size=seg * len(seg_scales), dtype=np.uint8)
    codes[(codes & 0x7F) == 0x7F] = 0x7E   # no NaN codes (the reference throws on them)
    for i in range(len(seg_scales)):       # each sender's chunk reached 448 (its own amax)
        codes[i * seg + 5] = 0x7E
    if seg_scales == [1.0, 1.0]:
        codes[:] = rng.choice(np.array([0x00, 0x80], np.uint8), size=codes.size)
    sc = np.array(seg_scales, np.float32)
    x = np.concatenate([R.dequantize(codes[i * seg:(i + 1) * seg], sc[i]) for i in range(len(sc))])
    want, ws = R.quantize(x)
    q = fu.requantize(T(codes, torch.uint8), T(sc, torch.float32), seg)
    assert q.scale == ws
    got = q.codes.cpu().numpy()
    bad = np.flatnonzero(got != want)
    assert bad.size == 0, (bad[:5], got[bad[:5]], want[bad[:5]])
    # the hop after: same values, one scale -> the codes come back unchanged
    q2 = fu.requantize(q.codes, q.scale_dev, q.codes.numel())
    want2, ws2 = R.quantize(R.dequantize(got, np.float32(q.scale)))
    assert q2.scale == ws2 and np.array_equal(q2.codes.cpu().numpy(), want2)


@pytest.mark.parametrize("shape", [(1, 3, 576, 128), (1, 24, 576, 128), (1, 24, 2304, 128),
                                   (1, 24, 6912, 128)])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_quantize_one_launch_and_two_pass_bit_exact(cuda, fu, shape, dtype):
    # per-tensor quantize: tensors that fit the grid's registers take the one-launch
    # cooperative kernel (quantize_fused_kernel), larger ones the two dependent passes; both
    # bit-exact vs the reference quantizer (fp8.cpp:107-123), twice in a row (the barrier and
    # amax words must be left zero)
    rng = np.random.default_rng(sum(shape))
    x = rng.uniform(-2.5, 2.5, size=shape).astype(np.float32)
    x.ravel()[::97] *= np.float32(1e-5)          # the E4M3 subnormal range (exact division)
    xt = T(x, dtype)
    want, ws = R.quantize(xt.float().cpu().numpy())
    for _ in range(2):
        n0 = fu.kernel_launch_count()
        q = fu.quantize(xt, check_finite=False)
        launches = fu.kernel_launch_count() - n0
        assert q.scale == ws
        got = q.codes.cpu().numpy().reshape(-1)
        bad = np.flatnonzero(got != want.reshape(-1))
        assert bad.size == 0, (bad[:5], got[bad[:5]], want.reshape(-1)[bad[:5]])
    nbytes = x.size * (2 if dtype == torch.bfloat16 else 4)
    if nbytes <= 4 << 20:       # well inside one resident wave's registers: one launch
        assert launches == 1, launches
    elif nbytes >= 30 << 20:    # beyond them: the two dependent passes
        assert launches == 2, launches

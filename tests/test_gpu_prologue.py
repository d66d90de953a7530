"""GPU parity of the fused QK RMSNorm + RoPE prologue (fusp_usp_attention_ex).

The reference's usp_attention takes Q/K after normalization and rotation, so the oracle is
restate.qk_prologue (float64 textbook definition) followed by the reference algorithm
(restate.attention_with_lse / restate.usp_attention).  The product writes the normalized rows
in the tensor cores' dtype (bf16; f16 for Q on the FP8 path) straight into the all-to-all
slots, so the oracle rounds Q'/K' the same way; the FP8 path quantizes K' from f32.
Bars: rel-L2 <= 1e-3 (bf16) and <= 2e-3 against the oracle's own FP8 output."""
import numpy as np
import pytest
import torch

from oracle import restate as R
from oracle.make_golden import qkv

pytestmark = pytest.mark.gpu

D = 128
EPS = 1e-6


def rel_l2(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def tables(s, theta=10000.0):
    inv = theta ** (-np.arange(0, D, 2, dtype=np.float64) / D)
    ang = np.arange(s, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)


def weights(seed):
    return R.rng_uniform(seed, D, 0.5, 1.5).astype(np.float32)


def run(fu, q, k, v, n, r, pro, fp8=False, per_block=False):
    qs, ks, vs = ([torch.from_numpy(np.ascontiguousarray(s)).cuda().to(torch.bfloat16)
                   for s in R.split_sequence(t, n)] for t in (q, k, v))
    mesh = fu.make_mesh(n, r)
    opts = fu.CommOptions(fp8_kv=fp8, fp8_block=per_block)
    rep = fu.run_protocol(n, lambda ctx: fu.usp_attention(
        ctx, qs[ctx.rank()], ks[ctx.rank()], vs[ctx.rank()], mesh, opts, prologue=pro))
    return torch.cat([o.float() for o in rep.results], dim=2).cpu().numpy()


def make_pro(fu, qw, kw, cos, sin):
    t = (lambda a: None if a is None else torch.from_numpy(a).cuda().contiguous())
    return fu.QKPrologue(q_norm_weight=t(qw), k_norm_weight=t(kw), eps=EPS, rope_cos=t(cos),
                         rope_sin=t(sin))


def oracle_qk(q, k, qw, kw, cos, sin, q_round, k_round):
    qp = q_round(R.qk_prologue(q, qw, EPS, cos, sin))
    kp = k_round(R.qk_prologue(k, kw, EPS, cos, sin))
    return qp, kp


def round_f16(x):
    return np.asarray(x, np.float32).astype(np.float16).astype(np.float32)


def f32(x):
    return np.asarray(x, np.float32)


@pytest.mark.parametrize("n,r", [(1, 1), (2, 1), (2, 2), (4, 2), (8, 2), (4, 4)])
@pytest.mark.parametrize("parts", ["norm_rope", "norm", "rope"])
def test_prologue_usp_bf16(cuda, fu, n, r, parts):
    h, s = 8, 128 * n
    q, k, v = qkv((1, h, s, D), (1, h, s, D), seeds=(21, 22, 23), lo=-2, hi=2)
    qw, kw = (weights(31), weights(32)) if "norm" in parts else (None, None)
    cos, sin = tables(s) if "rope" in parts else (None, None)
    out = run(fu, q, k, v, n, r, make_pro(fu, qw, kw, cos, sin))
    qp, kp = oracle_qk(q, k, qw, kw, cos, sin, R.round_bf16, R.round_bf16)
    want, _ = R.attention_with_lse(qp, kp, v)
    assert rel_l2(out, want) <= 1e-3


@pytest.mark.parametrize("n,r", [(1, 1), (2, 1), (2, 2), (4, 2)])
@pytest.mark.parametrize("per_block", [False, True])
def test_prologue_usp_fp8(cuda, fu, n, r, per_block):
    h, s = 8, 128 * n
    q, k, v = qkv((1, h, s, D), (1, h, s, D), seeds=(24, 25, 26), lo=-2, hi=2)
    qw, kw = weights(33), weights(34)
    cos, sin = tables(s)
    out = run(fu, q, k, v, n, r, make_pro(fu, qw, kw, cos, sin), fp8=True, per_block=per_block)
    qp, kp = oracle_qk(q, k, qw, kw, cos, sin, round_f16, f32)
    want = R.usp_attention(qp, kp, v, n, r, fp8=True, per_block=per_block)
    assert rel_l2(out, want) <= 2e-3


def test_prologue_explicit_positions(cuda, fu):
    """rope_pos0 shifts the table rows: a world-1 layer at offset 64 == rows 64.. of the table."""
    q, k, v = qkv((1, 4, 128, D), (1, 4, 128, D), seeds=(27, 28, 29))
    cos, sin = tables(256)
    pro = make_pro(fu, None, None, cos, sin)
    pro.rope_pos0 = 64
    out = run(fu, q, k, v, 1, 1, pro)
    qp = R.round_bf16(R.rope_interleaved(q, cos, sin, 64))
    kp = R.round_bf16(R.rope_interleaved(k, cos, sin, 64))
    want, _ = R.attention_with_lse(qp, kp, v)
    assert rel_l2(out, want) <= 1e-3


def test_prologue_errors(cuda, fu):
    q, k, v = qkv((1, 4, 128, D), (1, 4, 128, D))
    cos, sin = tables(64)  # too short for 128 positions
    with pytest.raises(fu.ShapeError, match="rope table"):
        run(fu, q, k, v, 1, 1, make_pro(fu, None, None, cos, sin))
    cos, sin = tables(128)
    pro = make_pro(fu, None, None, cos, sin)
    pro.rope_sin = None
    with pytest.raises(fu.InvalidArgument, match="go together"):
        run(fu, q, k, v, 1, 1, pro)


def test_prologue_is_one_launch_per_operand(cuda, fu):
    """The prologue replaces the pack: the layer launches no more kernels with it than
    without it (U > 1, bf16)."""
    q, k, v = qkv((1, 8, 256, D), (1, 8, 256, D))
    cos, sin = tables(256)
    pro = make_pro(fu, weights(1), weights(2), cos, sin)
    run(fu, q, k, v, 2, 1, None)
    torch.cuda.synchronize()
    c0 = fu.kernel_launch_count()
    run(fu, q, k, v, 2, 1, None)
    torch.cuda.synchronize()
    c1 = fu.kernel_launch_count()
    run(fu, q, k, v, 2, 1, pro)
    torch.cuda.synchronize()
    c2 = fu.kernel_launch_count()
    assert c2 - c1 == c1 - c0

"""GPU: head dims other than 128 (the reference's attention_core is generic in D,
tensor.cpp:143-181; SPEC.md's parity grids use small D).  D = 128 runs on the tcgen05 kernel;
any other D that is a multiple of 8 (up to 256) runs on attention_generic.cu's f32 CUDA-core
kernel, through the same protocols (Ulysses reshards, ring merge, FP8 wire, LSE, reshards)."""
import numpy as np
import pytest
import torch

from oracle import ref, ref_available
from oracle import restate as R

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_ref():
    if not ref_available():
        pytest.skip("oracle/_ref not built")


def rel_l2(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def qkv(shape, seeds=(111, 112, 113)):
    return [R.rng_tensor(s, shape).astype(np.float32) for s in seeds]


@pytest.mark.parametrize("d", [8, 16, 64, 256])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_attention_with_lse_other_head_dims(cuda, fu, d, dtype):
    q, k, v = qkv((1, 3, 100, d))
    if dtype == torch.bfloat16:
        q, k, v = R.round_bf16(q), R.round_bf16(k), R.round_bf16(v)
    want_o, want_l = ref.attention_with_lse(q, k, v)
    res = fu.attention_with_lse(*(torch.from_numpy(x).cuda().to(dtype) for x in (q, k, v)))
    assert rel_l2(res.out.cpu().numpy(), want_o) <= 1e-5
    assert np.abs(res.lse.cpu().numpy() - want_l).max() <= 1e-5


@pytest.mark.parametrize("d", [8, 64])
@pytest.mark.parametrize("n,r", [(4, 2), (4, 1), (4, 4), (8, 2)])
@pytest.mark.parametrize("fp8", [False, True])
def test_usp_other_head_dims_vs_reference(cuda, fu, d, n, r, fp8):
    # f32 inputs: the generic kernel computes in f32 like the reference (FP8: against the
    # reference's own FP8 path, same wire bytes)
    h, s = 8, 16 * n
    q, k, v = qkv((1, h, s, d))
    want, a2a, snd = ref.usp_attention(q, k, v, n, r, fp8=fp8, traffic=True)
    qs, ks, vs = ([torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in R.split_sequence(t, n)]
                  for t in (q, k, v))
    mesh = fu.make_mesh(n, r)
    opts = fu.CommOptions(fp8_kv=fp8, pipelined_ring=True)
    rep = fu.run_protocol(n, lambda ctx: fu.usp_attention(ctx, qs[ctx.rank()], ks[ctx.rank()],
                                                          vs[ctx.rank()], mesh, opts))
    got = torch.cat(rep.results, dim=2).cpu().numpy()
    assert rel_l2(got, want) <= (1e-4 if fp8 else 1e-5)
    assert [t[0] for t in rep.traffic] == [int(x) for x in a2a]  # the reference's own bytes
    assert [t[1] for t in rep.traffic] == [int(x) for x in snd]


def test_head_dim_errors(cuda, fu):
    x = torch.zeros(1, 2, 16, 12, device="cuda")
    with pytest.raises(fu.ShapeError, match="head dim D=12 unsupported"):
        fu.attention_with_lse(x, x, x)
    y = torch.zeros(1, 2, 16, 64, device="cuda")
    with pytest.raises(fu.ShapeError, match="qk prologue: head dim must be 128"):
        fu.run_protocol(1, lambda ctx: fu.usp_attention(ctx, y, y, y, fu.make_mesh(1, 1),
                                                        prologue=fu.QKPrologue(eps=1e-6)))

"""GPU parity of the persistent attention kernel's two work schedules.

"whole" gives each CTA complete 256-row q-blocks; "split" (stream-K) cuts q-blocks into KV
segments owned by consecutive CTAs and merges the partial (O, m, l) in the last-arriving CTA.
"kv2" runs whole 128-row Q tiles on attn_kv2_kernel (the two softmax warpgroups split the KV
range and merge in the CTA); "kv2split" adds stream-K segments over those tiles.
Both must match the fp32 oracle (attention_core, tensor.cpp:143-202) at the north-star bar
(rel-L2 <= 1e-3 on O, |dLSE| <= 1e-4), be deterministic run to run, and leave the ticket
counters clean for the next launch (any grid, any shape)."""
import numpy as np
import pytest
import torch

from oracle import restate as R
from oracle.make_golden import qkv

pytestmark = pytest.mark.gpu

REL_L2 = 1e-3
LSE_TOL = 1e-4


def rel_l2(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def T(x, dtype=torch.bfloat16):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda().to(dtype)


def run(fu, q, k, v, mode, ctas, out_dtype=torch.float32):
    with fu.attention_schedule(mode, ctas):
        r = fu.attention_with_lse(T(q), T(k), T(v), out_dtype=out_dtype)
        torch.cuda.synchronize()
    return r.out.float().cpu().numpy(), r.lse.cpu().numpy()


# (h, sq, skv, max_ctas): one q-block cut into many segments, ragged rows/keys, the FLUX
# per-rank shapes of the USP meshes, grids that do not divide the work.
CASES = [
    (1, 256, 4608, 0),    # 1 q-block x 36 tiles over 18 CTAs: 18 segments
    (1, 256, 4608, 7),
    (2, 300, 517, 3),     # ragged rows and keys
    (3, 512, 1000, 5),
    (3, 1024, 4608, 13),
    (6, 768, 2048, 148),
]


@pytest.mark.parametrize("h,sq,skv,ctas", CASES)
@pytest.mark.parametrize("mode", ["whole", "split", "auto", "kv2", "kv2split"])
def test_schedules_match_reference(cuda, fu, h, sq, skv, ctas, mode):
    q, k, v = qkv((1, h, sq, 128), (1, h, skv, 128), seeds=(11, 12, 13))
    ro, rl = R.attention_with_lse(q, k, v)
    o, l = run(fu, q, k, v, mode, ctas)
    assert rel_l2(o, ro) <= REL_L2
    assert np.abs(l - rl).max() <= LSE_TOL


@pytest.mark.parametrize("mode", ["split", "kv2split"])
def test_split_deterministic_and_counters_clean(cuda, fu, mode):
    q, k, v = qkv((1, 3, 1024, 128), (1, 3, 4608, 128), seeds=(1, 2, 3))
    a = run(fu, q, k, v, mode, 11)
    # a different grid and shape in between must not see stale tickets
    q2, k2, v2 = qkv((1, 1, 256, 128), (1, 1, 2048, 128), seeds=(4, 5, 6))
    ro2, _ = R.attention_with_lse(q2, k2, v2)
    for ctas in (3, 16, 0):
        for m2 in ("split", "kv2split"):
            o2, _ = run(fu, q2, k2, v2, m2, ctas)
            assert rel_l2(o2, ro2) <= REL_L2
    b = run(fu, q, k, v, mode, 11)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    w = run(fu, q, k, v, "whole", 0)
    assert rel_l2(a[0], w[0]) <= 4e-4  # two roundings of the same sums (each ~2e-4 from fp64)


def test_split_flux_u8_rank_shape(cuda, fu):
    # FLUX at Ulysses 8: one rank attends 3 heads x 4608 rows (54 q-blocks on 148 SMs)
    q, k, v = qkv((1, 3, 4608, 128), (1, 3, 4608, 128))
    o, l = run(fu, q, k, v, "auto", 0, out_dtype=torch.float16)
    rows = slice(0, 512)
    ro, rl = R.attention_with_lse(q[:, :, rows], k, v)
    assert rel_l2(o[:, :, rows], ro) <= REL_L2
    assert np.abs(l[:, :, rows] - rl).max() <= LSE_TOL
    w, wl = run(fu, q, k, v, "whole", 0, out_dtype=torch.float16)
    assert rel_l2(o, w) <= 1e-3
    assert np.abs(l - wl).max() <= 1e-5
    s, sl = run(fu, q, k, v, "kv2split", 0, out_dtype=torch.float16)
    assert rel_l2(s, w) <= 1e-3
    assert np.abs(sl - wl).max() <= 1e-5


@pytest.mark.parametrize("n,r", [(2, 2), (4, 4), (8, 2)])
def test_split_inside_ring_merge(cuda, fu, n, r):
    # ring steps >= 1 fuse merge_lse into the epilogue: the stream-K finisher must too
    q, k, v = qkv((1, 4, 256 * n, 128), (1, 4, 256 * n, 128), seeds=(21, 22, 23))
    full, _ = R.attention_with_lse(q, k, v)
    qs, ks, vs = ([torch.from_numpy(x).cuda().bfloat16() for x in R.split_sequence(t, n)]
                  for t in (q, k, v))
    mesh = fu.make_mesh(n, r)
    for mode in ("split", "whole", "kv2split"):
        with fu.attention_schedule(mode, 5):
            rep = fu.run_protocol(n, lambda ctx: fu.usp_attention(
                ctx, qs[ctx.rank()], ks[ctx.rank()], vs[ctx.rank()], mesh,
                fu.CommOptions(pipelined_ring=True)))
        out = torch.cat(rep.results, dim=2).cpu().numpy()
        assert rel_l2(out, full) <= REL_L2, mode

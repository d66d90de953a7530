"""GPU: the rest of the reference's protocol roster through the C ABI (protocols.hpp:28-95).

* LSE out of usp_attention / ulysses_attention (fusp_usp_attention_lse, the LSE riding a
  second all-to-all; the reference drops it at protocols.cpp:339, so the bar is the full
  attention's LSE from the oracle);
* ulysses / ring protocols over caller ProcessGroups that are not the world
  (fusp_group_create; protocols.hpp:47-65);
* detail::ulysses_input_reshard / ulysses_output_reshard (protocols.hpp:77-86): data movement
  and exact FP8 dequantization, bit-identical to the reference library."""
import numpy as np
import pytest
import torch

from oracle import ref, ref_available
from oracle import restate as R
from oracle.make_golden import qkv

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def shards(x, n, dtype=torch.bfloat16):
    return [torch.from_numpy(np.ascontiguousarray(s)).cuda().to(dtype) for s in R.split_sequence(x, n)]


@pytest.mark.parametrize("n,r,b", [(4, 2, 1), (4, 1, 1), (4, 1, 2), (8, 2, 2), (2, 2, 1)])
def test_usp_attention_returns_lse(cuda, fu, n, r, b):
    q, k, v = qkv((b, 8, 64 * n, 128), (b, 8, 64 * n, 128), seeds=(11, 12, 13))
    full_o, full_l = R.attention_with_lse(q, k, v)
    qs, ks, vs = shards(q, n), shards(k, n), shards(v, n)
    mesh = fu.make_mesh(n, r)
    opts = fu.CommOptions(pipelined_ring=True)
    rep = fu.run_protocol(n, lambda ctx: (
        fu.usp_attention_with_lse(ctx, qs[ctx.rank()], ks[ctx.rank()], vs[ctx.rank()], mesh, opts),
        fu.usp_attention(ctx, qs[ctx.rank()], ks[ctx.rank()], vs[ctx.rank()], mesh, opts)))
    out = torch.cat([x[0].out for x in rep.results], dim=2).cpu().numpy()
    lse = torch.cat([x[0].lse for x in rep.results], dim=2).cpu().numpy()
    assert rel_l2(out, full_o) <= 1e-3
    assert np.abs(lse - full_l).max() <= 1e-4
    for a, plain in rep.results:  # asking for the LSE does not change the output
        assert torch.equal(a.out, plain)


def test_ulysses_return_lse(cuda, fu):
    q, k, v = qkv((1, 8, 256, 128), (1, 8, 256, 128), seeds=(14, 15, 16))
    full_o, full_l = R.attention_with_lse(q, k, v)
    qs, ks, vs = shards(q, 4), shards(k, 4), shards(v, 4)
    rep = fu.run_protocol(4, lambda ctx: fu.ulysses_attention(
        ctx, qs[ctx.rank()], ks[ctx.rank()], vs[ctx.rank()], return_lse=True))
    assert rel_l2(torch.cat([x.out for x in rep.results], 2).cpu().numpy(), full_o) <= 1e-3
    assert np.abs(torch.cat([x.lse for x in rep.results], 2).cpu().numpy() - full_l).max() <= 1e-4


@pytest.mark.parametrize("fp8", [False, True])
def test_subgroup_protocols(cuda, fu, fp8):
    # a 4-rank world split into two disjoint groups that each run their own problem
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    probs = [qkv((1, 4, 128, 128), (1, 4, 128, 128), seeds=(s, s + 1, s + 2)) for s in (21, 31)]
    uly_groups = [[0, 1], [2, 3]]
    ring_groups = [[3, 1], [2, 0]]  # not in rank order: positions follow the member list

    def where(groups, rank):
        for gi, g in enumerate(groups):
            if rank in g:
                return gi, g.index(rank)

    parts = [[shards(t, 2) for t in p] for p in probs]
    opts = fu.CommOptions(fp8_kv=fp8)

    def prog(ctx):
        gi, pos = where(uly_groups, ctx.rank())
        grp = fu.ProcessGroup(uly_groups[gi])
        u = fu.ulysses_attention(ctx, *(t[pos] for t in parts[gi]), group=grp, opts=opts)
        gi, pos = where(ring_groups, ctx.rank())
        grp = fu.ProcessGroup(ring_groups[gi])
        rp = fu.ring_attention_pipelined(ctx, *(t[pos] for t in parts[gi]), group=grp, opts=opts)
        rs = fu.ring_attention_serial(ctx, *(t[pos] for t in parts[gi]), group=grp, opts=opts)
        return u, rp, rs

    rep = fu.run_protocol(4, prog)
    bar = 2e-3 if fp8 else 1e-3
    for gi, g in enumerate(uly_groups):
        got = torch.cat([rep.results[m][0] for m in g], dim=2).cpu().numpy()
        want = ref.ulysses_attention(*probs[gi], 2, fp8=fp8)
        assert rel_l2(got, want) <= bar
    for gi, g in enumerate(ring_groups):
        got = torch.cat([rep.results[m][1].out for m in g], dim=2).cpu().numpy()
        lse = torch.cat([rep.results[m][1].lse for m in g], dim=2).cpu().numpy()
        want_o, want_l = ref.ring_attention(*probs[gi], 2, fp8=fp8, pipelined=True)
        assert rel_l2(got, want_o) <= bar
        assert np.abs(lse - want_l).max() <= (2e-3 if fp8 else 1e-4)
        for m in g:  # serial == pipelined, bit for bit (protocols.hpp:60-62)
            assert torch.equal(rep.results[m][1].out, rep.results[m][2].out)


def test_group_errors_match_reference(cuda, fu):
    x = torch.zeros(1, 4, 16, 128, device="cuda")
    with pytest.raises(fu.FabricError, match=r"rank 0 not in group 1,2"):
        fu.run_protocol(4, lambda ctx: fu.ulysses_attention(ctx, x, x, x, group=fu.ProcessGroup([1, 2]))
                        if ctx.rank() == 0 else None)
    with pytest.raises(fu.FabricError, match=r"duplicate member 1 in group 1,1"):
        fu.run_protocol(2, lambda ctx: ctx.create_group([1, 1]))
    with pytest.raises(fu.FabricError, match=r"group member 5 out of range \[0,2\)"):
        fu.run_protocol(2, lambda ctx: ctx.create_group([0, 5]))


@pytest.mark.parametrize("n", [1, 2, 4])
@pytest.mark.parametrize("fp8", [False, True])
def test_reshards_bit_exact_vs_reference(cuda, fu, n, fp8):
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    q, k, v = qkv((1, 8, 32 * n, 128), (1, 8, 32 * n, 128), seeds=(41, 42, 43))
    want = ref.ulysses_input_reshard(q, k, v, n, fp8=fp8)  # [n][B, H/n, S, D] per rank
    qs, ks, vs = shards(q, n, torch.float32), shards(k, n, torch.float32), shards(v, n, torch.float32)

    def prog(ctx):
        rs = fu.detail.ulysses_input_reshard(ctx, qs[ctx.rank()], ks[ctx.rank()], vs[ctx.rank()],
                                             opts=fu.CommOptions(fp8_kv=fp8))
        back = fu.detail.ulysses_output_reshard(ctx, rs.q)
        return rs, back

    rep = fu.run_protocol(n, prog)
    for rank, (rs, back) in enumerate(rep.results):
        for got, w in zip((rs.q, rs.k, rs.v), want):
            assert np.array_equal(got.cpu().numpy(), w[rank])
        assert torch.equal(back, qs[rank])  # output reshard inverts the Q reshard exactly

"""GPU: the peer-memory Ulysses transport (fusp_ctx_peer_enable, csrc/peer.cu).

With peer windows the two Ulysses reshards of a USP layer (protocols.cpp:125-203) are fused into
the kernels around them: the pack kernel stores every member's slot straight into that member's
window, the attention epilogue stores O / LSE rows straight into their owner's window, and one
signal-and-wait kernel per reshard replaces the all-to-all.  Ranks are threads on cuda:0 here (a
window of another rank is then plain device memory: the same kernels and the same protocol as
over NVLink).  The transport must not change a single bit: outputs, LSE and TrafficLog bytes are
compared with the same layer over the in-process fabric, and with the reference's output."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from oracle import restate as R
from oracle.make_golden import qkv

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def shards(x, n, dtype=torch.bfloat16):
    return [torch.from_numpy(np.ascontiguousarray(s)).cuda().to(dtype) for s in R.split_sequence(x, n)]


def rel_l2(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def window(fu, n, r, sl, h=8, opts=None):
    return fu.peer_window_bytes(n, r, (1, h, sl, 128), torch.bfloat16, opts)


def layer(fu, qs, ks, vs, mesh, opts, peer_bytes=0, lse=False):
    """One USP layer per rank; per rank (output or (out, lse), traffic, peer stats)."""
    def prog(ctx):
        if peer_bytes:
            ctx.enable_peer_memory(peer_bytes)
        q, k, v = qs[ctx.rank()], ks[ctx.rank()], vs[ctx.rank()]
        if lse:
            a = fu.usp_attention_with_lse(ctx, q, k, v, mesh, opts)
            out = (a.out.clone(), a.lse.clone())
        else:
            out = fu.usp_attention(ctx, q, k, v, mesh, opts).clone()
        ctx.synchronize()
        return [out], ctx.traffic(), ctx.peer_stats() if peer_bytes else None
    return fu.run_protocol(len(qs), prog)


@pytest.mark.parametrize("n,r,fp8,block", [(2, 1, False, 0), (4, 1, False, 0), (8, 1, False, 0),
                                           (4, 2, False, 0), (8, 2, False, 0), (4, 1, True, 0),
                                           (8, 1, True, 1), (8, 4, True, 0)])
def test_peer_usp_bit_identical_to_fabric(cuda, fu, n, r, fp8, block):
    h, s = 8, 128 * n
    q, k, v = qkv((1, h, s, 128), (1, h, s, 128), seeds=(200 + n, 201 + r, 202 + int(fp8)))
    qs, ks, vs = shards(q, n), shards(k, n), shards(v, n)
    mesh = fu.make_mesh(n, r)
    opts = fu.CommOptions(fp8_kv=fp8, fp8_block=block, pipelined_ring=True, check_finite=False,
                          out_dtype=torch.float32)
    ref = layer(fu, qs, ks, vs, mesh, opts)
    got = layer(fu, qs, ks, vs, mesh, opts, peer_bytes=window(fu, n, r, s // n, h, opts))
    for a, b in zip(got.results, ref.results):
        assert torch.equal(a[0][0], b[0][0])
        assert a[1] == b[1]                   # TrafficLog bytes: the transport is invisible
        assert a[2] == (1, 0) if n // r > 1 else True  # the layer took the peer path
    out = torch.cat([x[0][0] for x in got.results], dim=2).cpu().numpy()
    want = R.usp_attention(q, k, v, n, r, fp8=True, per_block=bool(block)) if fp8 \
        else R.attention_with_lse(q, k, v)[0]
    assert rel_l2(out, want) <= (2e-3 if fp8 else 1e-3)


def test_peer_lse_and_output_dtypes(cuda, fu):
    n, h, s = 4, 8, 512
    q, k, v = qkv((1, h, s, 128), (1, h, s, 128), seeds=(211, 212, 213))
    qs, ks, vs = shards(q, n), shards(k, n), shards(v, n)
    mesh = fu.make_mesh(n, 1)
    for odt in (torch.float16, torch.bfloat16, torch.float32):
        opts = fu.CommOptions(check_finite=False, out_dtype=odt)
        ref = layer(fu, qs, ks, vs, mesh, opts, lse=True)
        got = layer(fu, qs, ks, vs, mesh, opts, peer_bytes=window(fu, n, 1, s // n, h, opts), lse=True)
        for a, b in zip(got.results, ref.results):
            assert torch.equal(a[0][0][0], b[0][0][0]) and torch.equal(a[0][0][1], b[0][0][1])


def test_peer_batch2(cuda, fu):
    # B > 1: the output region is [member][B][hp][SL][D] and is concatenated over heads
    n, h, s = 4, 8, 256
    q, k, v = qkv((2, h, s, 128), (2, h, s, 128), seeds=(221, 222, 223))
    qs, ks, vs = shards(q, n), shards(k, n), shards(v, n)
    mesh = fu.make_mesh(n, 1)
    opts = fu.CommOptions(check_finite=False, out_dtype=torch.float32)
    wb = fu.peer_window_bytes(n, 1, (2, h, s // n, 128), torch.bfloat16, opts)
    ref = layer(fu, qs, ks, vs, mesh, opts, lse=True)
    got = layer(fu, qs, ks, vs, mesh, opts, peer_bytes=wb, lse=True)
    for a, b in zip(got.results, ref.results):
        assert torch.equal(a[0][0][0], b[0][0][0]) and torch.equal(a[0][0][1], b[0][0][1])
        assert a[2] == (1, 0)


@pytest.mark.parametrize("r,fp8", [(1, False), (2, False), (4, True)])
def test_peer_back_to_back_layers_no_buffer_race(cuda, fu, r, fp8):
    # single-buffered windows: consecutive layers reuse every member's regions; a rank that
    # runs ahead must never overwrite data a slower member has not consumed (peer.cu header).
    # 12 layers with different inputs per layer, 8 ranks racing on one GPU; with R > 1 the
    # ring's hops go through the windows too (two receive buffers per rank, released to the
    # previous member once consumed -- within a layer and across layers).
    n, h, s = 8, 8, 1024
    probs = [qkv((1, h, s, 128), (1, h, s, 128), seeds=(300 + i, 400 + i, 500 + i)) for i in range(3)]
    per = [[shards(t, n) for t in p] for p in probs]
    mesh = fu.make_mesh(n, r)
    opts = fu.CommOptions(fp8_kv=fp8, pipelined_ring=True, check_finite=False, out_dtype=torch.float16)
    wb = window(fu, n, r, s // n, h, opts)

    def prog(peer):
        def body(ctx):
            if peer:
                ctx.enable_peer_memory(wb)
            outs = []
            for i in range(12):
                q, k, v = (t[ctx.rank()] for t in per[i % 3])
                outs.append(fu.usp_attention(ctx, q, k, v, mesh, opts).clone())
            ctx.synchronize()
            return outs, ctx.peer_stats() if peer else None
        return fu.run_protocol(n, body)

    ref, got = prog(False), prog(True)
    for a, b in zip(got.results, ref.results):
        assert a[1] == (12, 0)
        for x, y in zip(a[0], b[0]):
            assert torch.equal(x, y)


def test_peer_other_group_falls_back(cuda, fu):
    # the windows serve the first group they were used with; a layer over another group goes
    # through the fabric (counted), still correct
    n, h, s = 4, 4, 256
    q, k, v = qkv((1, h, s, 128), (1, h, s, 128), seeds=(231, 232, 233))
    full = shards(q, n), shards(k, n), shards(v, n)
    halves = [shards(t, 2) for t in (q, k, v)]
    mesh = fu.make_mesh(n, 1)
    opts = fu.CommOptions(check_finite=False)
    wb = window(fu, n, 1, s // n, h, opts)

    def prog(ctx):
        ctx.enable_peer_memory(wb)
        a = fu.usp_attention(ctx, *(t[ctx.rank()] for t in full), mesh, opts)
        g = [0, 1] if ctx.rank() < 2 else [2, 3]
        ctx.create_group(g)
        b = fu.ulysses_attention(ctx, *(t[g.index(ctx.rank())] for t in halves), group=fu.ProcessGroup(g))
        ctx.synchronize()
        return a, b, ctx.peer_stats()

    rep = fu.run_protocol(n, prog)
    want = R.attention_with_lse(q, k, v)[0]
    got = torch.cat([x[0].float() for x in rep.results], dim=2).cpu().numpy()
    assert rel_l2(got, want) <= 1e-3
    for m in (0, 2):
        sub = torch.cat([rep.results[m][1].float(), rep.results[m + 1][1].float()], dim=2).cpu().numpy()
        assert rel_l2(sub, want) <= 1e-3
    assert all(x[2] == (1, 1) for x in rep.results)


@pytest.mark.parametrize("r", [1])
def test_peer_graph_capture_multi_rank(cuda, fu, r):
    # a peer-path layer needs no host rendezvous -- the Ulysses reshards AND the ring's hops
    # (R > 1) go through the windows -- so it is capturable on in-process ranks (the fabric
    # path is not); 3 replays with new inputs each match eager
    n, h, s = 4, 8, 512
    mesh = fu.make_mesh(n, r)
    opts = fu.CommOptions(pipelined_ring=True, check_finite=False, out_dtype=torch.float16)
    wb = window(fu, n, r, s // n, h, opts)
    probs = [qkv((1, h, s, 128), (1, h, s, 128), seeds=(240 + i, 250 + i, 260 + i)) for i in range(3)]
    per = [[shards(t, n) for t in p] for p in probs]

    def prog(ctx):
        ctx.enable_peer_memory(wb)
        r = ctx.rank()
        q, k, v = (per[0][t][r].clone() for t in range(3))
        out = torch.empty_like(q, dtype=torch.float16)
        g = fu.LayerGraph(ctx, q[None], k[None], v[None], out[None], mesh, opts, 1)
        res = []
        for i in range(3):
            for dst, t in zip((q, k, v), range(3)):
                dst.copy_(per[i][t][r])
            g.launch()
            res.append(out.clone())
            eager = fu.usp_attention(ctx, per[i][0][r], per[i][1][r], per[i][2][r], mesh, opts)
            res.append(eager.clone())
        ctx.synchronize()
        g.close()
        return res

    rep = fu.run_protocol(n, prog)
    for r in rep.results:
        for i in range(3):
            assert torch.equal(r[2 * i], r[2 * i + 1])


def test_peer_stalled_member_raises_deadlock(cuda, fu):
    # a member that never joins: the exchange kernel's bounded spin sets the timeout flag and
    # fusp_ctx_synchronize raises DeadlockError instead of hanging (FUSP_TIMEOUT_S=3)
    code = r"""
import threading, torch, paper_2602_10940_b200 as fu
q = torch.randn(1, 4, 128, 128, device="cuda", dtype=torch.bfloat16)
mesh = fu.make_mesh(2, 1)
opts = fu.CommOptions(check_finite=False)
wb = fu.peer_window_bytes(2, 1, (1, 4, 128, 128))
done = threading.Event()
def prog(ctx):
    ctx.enable_peer_memory(wb)
    if ctx.rank() == 1:  # joins the setup, never the layer; keeps its window alive meanwhile
        done.wait(120)
        return "absent"
    try:
        fu.usp_attention(ctx, q, q, q, mesh, opts)
        ctx.synchronize()
    except fu.DeadlockError as e:
        return "DeadlockError: " + str(e)
    finally:
        done.set()
    return "no error"
print(fu.run_protocol(2, prog).results[0])
"""
    env = dict(os.environ, FUSP_TIMEOUT_S="3", PYTHONPATH=os.path.dirname(HERE))
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, env=env)
    assert "DeadlockError: deadlock: rank 0" in p.stdout, p.stdout + p.stderr[-2000:]


@pytest.mark.parametrize("n,r", [(2, 1), (4, 1), (8, 1), (4, 2), (8, 2)])
def test_peer_block_producer_and_consumer(cuda, fu, n, r):
    # fusp_usp_block on the peer path: the QKV projection's epilogue stores Q, K, V into the
    # members' windows (GEMM and input all-to-all in one kernel) and the output projection
    # reads O where the members' attention epilogues stored it (no copy-out).  Three blocks
    # back to back with different inputs (single-buffered windows reused); bit-identical to
    # the same blocks over the in-process fabric.
    heads, s, c, nout = 8, 256 * n, 256, 256
    rs = np.random.RandomState(70 + n + r)
    xs_all = [R.round_bf16(rs.uniform(-1, 1, (1, s, c)).astype(np.float32)) for _ in range(3)]
    wqkv = R.round_bf16((rs.uniform(-1, 1, (c, 3 * heads * 128)) / np.sqrt(c)).astype(np.float32))
    wout = R.round_bf16((rs.uniform(-1, 1, (heads * 128, nout)) / np.sqrt(heads * 128)).astype(np.float32))
    xs = [[torch.from_numpy(np.ascontiguousarray(t)).cuda().bfloat16() for t in np.split(x, n, axis=1)]
          for x in xs_all]
    wq_d, wo_d = torch.from_numpy(wqkv).cuda().bfloat16(), torch.from_numpy(wout).cuda().bfloat16()
    mesh = fu.make_mesh(n, r)
    opts = fu.CommOptions(check_finite=False)
    wb = fu.peer_window_bytes(n, r, (1, heads, s // n, 128), torch.bfloat16,
                              fu.CommOptions(check_finite=False, out_dtype=torch.bfloat16))

    def prog(peer):
        def body(ctx):
            if peer:
                ctx.enable_peer_memory(wb)
            ys = [fu.usp_block(ctx, xs[i][ctx.rank()], wq_d, heads, wo_d, mesh, opts=opts,
                               out_dtype=torch.float32).clone() for i in range(3)]
            ctx.synchronize()
            return ys, ctx.traffic(), ctx.peer_stats() if peer else None
        return fu.run_protocol(n, body)

    ref, got = prog(False), prog(True)
    for a, b in zip(got.results, ref.results):
        assert a[2] == (3, 0)       # every block's reshards took the peer path
        assert a[1] == b[1]         # same TrafficLog bytes
        for x, y in zip(a[0], b[0]):
            assert torch.equal(x, y)


def test_peer_refuses_shared_hardware_queues(cuda, fu):
    # ranks as threads on one device with too few hardware queues for their streams would wait
    # behind each other's spinning exchange kernels: enabling the windows fails loudly instead
    code = r'''
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2602_10940_b200 as fu
def prog(ctx):
    try:
        ctx.enable_peer_memory(1 << 20)
    except fu.FuspError as e:
        return str(e)
    return "enabled"
rep = fu.run_protocol(4, prog)
print("RESULTS", rep.results)
'''
    env = dict(os.environ, CUDA_DEVICE_MAX_CONNECTIONS="4")
    p = subprocess.run([sys.executable, "-c", code], cwd=os.path.dirname(HERE), env=env,
                       capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    line = [x for x in p.stdout.splitlines() if x.startswith("RESULTS")][0]
    assert line.count("CUDA_DEVICE_MAX_CONNECTIONS >= 8") == 4, line


@pytest.mark.parametrize("world,ring,fp8,graph,bsz", [(2, 1, 0, False, 1), (4, 2, 0, True, 1),
                                                      (4, 4, 1, True, 1), (4, 2, 1, False, 1),
                                                      (4, 2, 2, False, 1), (4, 2, 0, False, 2)])
def test_peer_windows_across_processes_ipc(cuda, fu, tmp_path, world, ring, fp8, graph, bsz):
    # PROCESSES on cuda:0, windows mapped through CUDA IPC (the deployment path: one process per
    # GPU) -- the pointer path of ranks-as-threads never opens an IPC handle.  Contexts of
    # different processes time-slice the GPU (separate hardware queues), so the spinning
    # exchanges see each other's signals slice by slice.  With R > 1 the ring's K / V hops go
    # through the windows too (copies into the next member's ring buffers, released back by
    # signals), and the three layers also run as ONE captured graph.  Outputs equal the
    # in-process layer over the fabric bit for bit.
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "peer_ipc_worker.py"), str(r),
                               str(world), str(tmp_path), str(ring), str(fp8), str(int(graph)), str(bsz)],
                              cwd=os.path.dirname(HERE), stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                              text=True, env=dict(os.environ, FUSP_TIMEOUT_S="60"))
             for r in range(world)]
    errs = [p.communicate(timeout=900)[1] for p in procs]
    assert all(p.returncode == 0 for p in procs), [e[-1500:] for e in errs]
    got = [torch.load(tmp_path / f"out{r}.pt") for r in range(world)]
    assert all(tuple(g["stats"])[0] >= 3 and tuple(g["stats"])[1] == 0 for g in got)
    h, s = 8, 256 * world
    mesh = fu.make_mesh(world, ring)
    opts = fu.CommOptions(fp8_kv=fp8 > 0, fp8_block=int(fp8 == 2), pipelined_ring=True,
                          check_finite=False, out_dtype=torch.float32)
    for i in range(3):
        q, k, v = qkv((bsz, h, s, 128), (bsz, h, s, 128), seeds=(600 + i, 610 + i, 620 + i))
        qs, ks, vs = shards(q, world), shards(k, world), shards(v, world)
        ref = layer(fu, qs, ks, vs, mesh, opts)
        for r in range(world):
            assert torch.equal(got[r]["outs"][i], ref.results[r][0][0].cpu())
            if graph:
                assert torch.equal(got[r]["gouts"][i], ref.results[r][0][0].cpu())
                if i == 0:  # the eager layer after the replays
                    assert torch.equal(got[r]["outs"][3], ref.results[r][0][0].cpu())


@pytest.mark.parametrize("n,fp8", [(1, False), (4, False), (1, True), (2, True)])
def test_block_graph_replays_match_eager(cuda, fu, n, fp8):
    # the whole MMDiT attention block (QKV projection -> USP layer -> output projection) of 3
    # layers captured as ONE CUDA graph (fusp_graph_capture_block), replayed with new inputs:
    # bit-identical to eager blocks.  n = 4: ranks as threads with peer windows -- the fused
    # producer / epilogue stores and the signal kernels inside the graph, no host rendezvous.
    heads, c, nout, layers = 8, 256, 256, 3
    s = 256 * n
    rs = np.random.RandomState(90 + n)
    w = R.round_bf16((rs.uniform(-1, 1, (c, 3 * heads * 128)) / np.sqrt(c)).astype(np.float32))
    wo = R.round_bf16((rs.uniform(-1, 1, (heads * 128, nout)) / np.sqrt(heads * 128)).astype(np.float32))
    w_d, wo_d = torch.from_numpy(w).cuda().bfloat16(), torch.from_numpy(wo).cuda().bfloat16()
    xs = [R.round_bf16(rs.uniform(-1, 1, (layers, 1, s, c)).astype(np.float32)) for _ in range(2)]
    mesh = fu.make_mesh(n, 1)
    # (FP8: the block stages Q, K, V and the layer quantizes K, V -- the two-pass form under
    # capture, the one-launch form eager: the same codes)
    opts = fu.CommOptions(fp8_kv=fp8, check_finite=False)
    wb = fu.peer_window_bytes(n, 1, (1, heads, s // n, 128), torch.bfloat16,
                              fu.CommOptions(fp8_kv=fp8, check_finite=False, out_dtype=torch.bfloat16))

    def prog(ctx):
        if n > 1:
            ctx.enable_peer_memory(wb)
        r = ctx.rank()
        part = [torch.from_numpy(np.ascontiguousarray(np.split(x, n, axis=2)[r])).cuda().bfloat16()
                for x in xs]
        xin = part[0].clone()
        y = torch.empty(layers, 1, s // n, nout, device="cuda", dtype=torch.float32)
        g = fu.BlockGraph(ctx, xin, w_d, heads, wo_d, y, mesh, opts=opts, layers=layers)
        res = []
        for p in part:
            xin.copy_(p)
            g.launch()
            got = y.clone()
            eager = torch.stack([fu.usp_block(ctx, p[i], w_d, heads, wo_d, mesh, opts=opts,
                                              out_dtype=torch.float32) for i in range(layers)])
            res.append((got, eager))
        ctx.synchronize()
        g.close()
        return res

    rep = fu.run_protocol(n, prog)
    for r in rep.results:
        for got, eager in r:
            assert torch.equal(got, eager)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float16])
@pytest.mark.parametrize("n,r,fp8", [(4, 1, False), (4, 2, False), (4, 1, True)])
def test_peer_input_dtypes_bit_identical(cuda, fu, dtype, n, r, fp8):
    # the wire carries the caller's dtype (f32 inputs put exactly the reference's bytes on it;
    # f16 as is) and the receiver stages the operands: through the windows as through the
    # fabric, bit for bit, with the reference's TrafficLog bytes
    h, s = 8, 128 * n
    q, k, v = qkv((1, h, s, 128), (1, h, s, 128), seeds=(700 + n, 701 + r, 702 + int(fp8)))
    qs, ks, vs = shards(q, n, dtype), shards(k, n, dtype), shards(v, n, dtype)
    mesh = fu.make_mesh(n, r)
    opts = fu.CommOptions(fp8_kv=fp8, pipelined_ring=True, check_finite=False, out_dtype=torch.float32)
    wb = fu.peer_window_bytes(n, r, (1, h, s // n, 128), dtype, opts)
    ref = layer(fu, qs, ks, vs, mesh, opts)
    got = layer(fu, qs, ks, vs, mesh, opts, peer_bytes=wb)
    for a, b in zip(got.results, ref.results):
        assert torch.equal(a[0][0], b[0][0])
        assert a[1] == b[1]
        assert a[2] == (1, 0)


def test_peer_check_finite_rejects_before_any_exchange(cuda, fu):
    # check_finite validates the local inputs before the pack (protocols.cpp:97-105): every rank
    # raises InvalidArgument with the reference's message and no rank is left in an exchange
    n, h, s = 4, 4, 512
    q, k, v = qkv((1, h, s, 128), (1, h, s, 128), seeds=(801, 802, 803))
    qs, ks, vs = shards(q, n), shards(k, n), shards(v, n)
    for t in ks:
        t[0, 0, 3, 5] = float("nan")
    mesh = fu.make_mesh(n, 1)
    opts = fu.CommOptions(check_finite=True)
    wb = window(fu, n, 1, s // n, h, opts)

    def prog(ctx):
        ctx.enable_peer_memory(wb)
        try:
            fu.usp_attention(ctx, qs[ctx.rank()], ks[ctx.rank()], vs[ctx.rank()], mesh, opts)
        except fu.InvalidArgument as e:
            msg = str(e)
        else:
            msg = "no error"
        # the windows still work afterwards (nothing half-exchanged)
        ok = fu.usp_attention(ctx, qs[ctx.rank()], qs[ctx.rank()], vs[ctx.rank()], mesh,
                              fu.CommOptions(check_finite=False))
        ctx.synchronize()
        return msg, bool(torch.isfinite(ok).all())

    rep = fu.run_protocol(n, prog)
    for msg, finite in rep.results:
        assert "non-finite" in msg and finite


@pytest.mark.parametrize("n,r,fp8", [(4, 1, False), (8, 2, False), (4, 1, True)])
def test_peer_qk_prologue_bit_identical(cuda, fu, n, r, fp8):
    # the fused QK RMSNorm + RoPE pack stores into the members' windows like the plain pack
    h, s = 8, 128 * n
    q, k, v = qkv((1, h, s, 128), (1, h, s, 128), seeds=(900 + n, 901 + r, 902 + int(fp8)))
    qs, ks, vs = shards(q, n), shards(k, n), shards(v, n)
    mesh = fu.make_mesh(n, r)
    cos, sin = fu.rope_tables(s)
    rs = np.random.RandomState(n + r)
    pro = fu.QKPrologue(q_norm_weight=torch.from_numpy(rs.uniform(0.5, 1.5, 128).astype(np.float32)).cuda(),
                        k_norm_weight=torch.from_numpy(rs.uniform(0.5, 1.5, 128).astype(np.float32)).cuda(),
                        eps=1e-6, rope_cos=cos, rope_sin=sin)
    opts = fu.CommOptions(fp8_kv=fp8, pipelined_ring=True, check_finite=False, out_dtype=torch.float32)
    wb = window(fu, n, r, s // n, h, opts)

    def run(peer):
        def prog(ctx):
            if peer:
                ctx.enable_peer_memory(wb)
            i = ctx.rank()
            out = fu.usp_attention(ctx, qs[i], ks[i], vs[i], mesh, opts, prologue=pro).clone()
            ctx.synchronize()
            return out, ctx.traffic(), ctx.peer_stats() if peer else None
        return fu.run_protocol(n, prog)

    ref, got = run(False), run(True)
    for a, b in zip(got.results, ref.results):
        assert torch.equal(a[0], b[0])
        assert a[1] == b[1]
        assert a[2] == (1, 0)

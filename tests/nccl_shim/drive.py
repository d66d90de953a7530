"""Runs fastusp's NCCL backend (NcclComm) at world > 1 with ranks as threads on one GPU, under
LD_PRELOAD=tests/nccl_shim/_build/libnccl_shim.so (test infrastructure, see nccl_shim.cpp).
Prints one JSON line per check; tests/test_gpu_nccl_shim.py runs it and asserts."""
from __future__ import annotations

import json
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_10940_b200 as fu  # noqa: E402
from oracle import restate as R  # noqa: E402
from oracle.make_golden import qkv  # noqa: E402


def emit(**kw):
    print(json.dumps(kw), flush=True)


def nccl_world(n, fn):
    """fn(ctx) on n threads, each with its own NCCL context on cuda:0 and its own stream."""
    uid = fu.WorkerContext.nccl_unique_id()
    res, err = [None] * n, [None] * n

    def body(r):
        try:
            torch.cuda.set_device(0)
            ctx = fu.WorkerContext.nccl(uid, n, r, 0)
            s = torch.cuda.Stream()
            try:
                with torch.cuda.stream(s):
                    res[r] = fn(ctx)
                s.synchronize()
            finally:
                ctx.close()
        except BaseException as e:  # noqa: BLE001 -- reported below
            err[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(n)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    return res, err


def shards(x, n):
    return [torch.from_numpy(np.ascontiguousarray(s)).cuda().bfloat16() for s in R.split_sequence(x, n)]


def rel_l2(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def usp_cases():
    h = 8
    for n, r, fp8, pipelined in [(2, 1, False, False), (2, 2, False, True), (4, 2, False, True),
                                 (4, 4, True, True), (4, 1, True, False), (4, 2, True, False)]:
        s = 64 * n
        q, k, v = qkv((1, h, s, 128), (1, h, s, 128), seeds=(61 + n, 62 + r, 63))
        qs, ks, vs = shards(q, n), shards(k, n), shards(v, n)
        mesh = fu.make_mesh(n, r)
        opts = fu.CommOptions(fp8_kv=fp8, pipelined_ring=pipelined, check_finite=True)

        def prog(ctx):
            o = fu.usp_attention(ctx, qs[ctx.rank()], ks[ctx.rank()], vs[ctx.rank()], mesh, opts)
            t = ctx.traffic()
            a = fu.usp_attention_with_lse(ctx, qs[ctx.rank()], ks[ctx.rank()], vs[ctx.rank()], mesh, opts)
            ctx.synchronize()
            return o, a, t

        res, err = nccl_world(n, prog)
        if any(e is not None for e in err):
            emit(check=f"usp_n{n}_r{r}_fp8{int(fp8)}", ok=False, error=repr([e for e in err if e][0]))
            continue
        got = torch.cat([x[0].float() for x in res], dim=2).cpu().numpy()
        lse = torch.cat([x[1].lse for x in res], dim=2).cpu().numpy()
        if fp8:
            want, bar = R.usp_attention(q, k, v, n, r, fp8=True), 2e-3
        else:
            want, bar = R.attention_with_lse(q, k, v)[0], 1e-3
        e = rel_l2(got, want)
        # the same layer over the in-process copy-engine fabric: identical kernels and data, so
        # the NCCL path must agree bit for bit (and put the same bytes on the wire)
        loc = fu.run_protocol(n, lambda ctx: (fu.usp_attention(
            ctx, qs[ctx.rank()], ks[ctx.rank()], vs[ctx.rank()], mesh, opts)))
        same = all(torch.equal(a[0], b) for a, b in zip(res, loc.results))
        traffic_nccl = [list(x[2]) for x in res]
        traffic_local = [list(t) for t in loc.traffic]
        full_l = R.attention_with_lse(q, k, v)[1]
        lse_err = float(np.abs(lse - full_l).max())
        lse_ok = lse_err <= (5e-2 if fp8 else 1e-4)
        emit(check=f"usp_n{n}_r{r}_fp8{int(fp8)}_pipe{int(pipelined)}",
             ok=bool(e <= bar and same and traffic_nccl == traffic_local and lse_ok),
             rel_l2=e, bit_identical_to_local=same, lse_maxabs=lse_err,
             traffic_nccl=traffic_nccl, traffic_local=traffic_local)


def subgroups():
    n = 4
    probs = [qkv((1, 4, 128, 128), (1, 4, 128, 128), seeds=(s, s + 1, s + 2)) for s in (71, 81)]
    parts = [[shards(t, 2) for t in p] for p in probs]
    groups = [[0, 1], [2, 3]]

    def prog(ctx):
        gi = 0 if ctx.rank() < 2 else 1
        ctx.create_group(groups[gi])  # collective over the world (one ncclCommSplit)
        pos = groups[gi].index(ctx.rank())
        out = fu.ulysses_attention(ctx, *(t[pos] for t in parts[gi]), group=fu.ProcessGroup(groups[gi]))
        ring = fu.ring_attention_pipelined(ctx, *(t[pos] for t in parts[gi]),
                                           group=fu.ProcessGroup(groups[gi]))
        torch.cuda.current_stream().synchronize()
        return out, ring

    res, err = nccl_world(n, prog)
    if any(e is not None for e in err):
        emit(check="subgroups", ok=False, error=repr([e for e in err if e][0]))
        return
    worst = 0.0
    for gi, g in enumerate(groups):
        want = R.attention_with_lse(*probs[gi])[0]
        for idx in (0, 1):
            got = torch.cat([res[m][idx] if idx == 0 else res[m][idx].out for m in g], dim=2)
            worst = max(worst, rel_l2(got.float().cpu().numpy(), want))
    emit(check="subgroups_ulysses_and_ring", ok=worst <= 1e-3, rel_l2=worst)


def dead_peer():
    # rank 1 never joins the layer's all-to-all: rank 0 must get DeadlockError, not hang
    q, k, v = qkv((1, 4, 128, 128), (1, 4, 128, 128), seeds=(91, 92, 93))
    qs, ks, vs = shards(q, 2), shards(k, 2), shards(v, 2)
    mesh = fu.make_mesh(2, 1)

    def prog(ctx):
        if ctx.rank() == 1:
            return "absent"
        try:
            fu.usp_attention(ctx, qs[0], ks[0], vs[0], mesh, fu.CommOptions(check_finite=False))
            ctx.synchronize(timeout_s=10)
        except fu.DeadlockError as e:
            first = str(e)
        else:
            return "no error"
        try:  # the communicators were aborted: later collectives fail fast
            fu.usp_attention(ctx, qs[0], ks[0], vs[0], mesh, fu.CommOptions(check_finite=False))
        except fu.FabricError as e:
            return ("DeadlockError", first, "then", str(e))
        return ("DeadlockError", first, "then no error")

    res, err = nccl_world(2, prog)
    r0 = res[0]
    ok = isinstance(r0, tuple) and r0[0] == "DeadlockError" and "deadlock: rank 0" in r0[1] \
        and len(r0) == 4 and "aborted" in r0[3]
    emit(check="dead_peer_deadlock_error", ok=bool(ok), result=repr(r0), error=repr(err))


def peer_cases():
    # peer-memory windows set up through NcclComm (handles all-gathered by grouped
    # ncclSend/ncclRecv): the Ulysses reshards bypass NCCL, the ring (R > 1) still uses it
    h = 8
    for n, r, fp8 in [(2, 1, False), (4, 1, True), (4, 2, False)]:
        s = 128 * n
        q, k, v = qkv((1, h, s, 128), (1, h, s, 128), seeds=(161 + n, 162 + r, 163))
        qs, ks, vs = shards(q, n), shards(k, n), shards(v, n)
        mesh = fu.make_mesh(n, r)
        opts = fu.CommOptions(fp8_kv=fp8, pipelined_ring=True, check_finite=False)
        wb = fu.peer_window_bytes(n, r, (1, h, s // n, 128), torch.bfloat16, opts)

        def prog(ctx):
            ctx.enable_peer_memory(wb)
            outs = [fu.usp_attention(ctx, qs[ctx.rank()], ks[ctx.rank()], vs[ctx.rank()], mesh, opts).clone()
                    for _ in range(3)]
            ctx.synchronize()
            return outs, ctx.traffic(), ctx.peer_stats()

        res, err = nccl_world(n, prog)
        if any(e is not None for e in err):
            emit(check=f"peer_n{n}_r{r}", ok=False, error=repr([e for e in err if e][0]))
            continue
        loc = fu.run_protocol(n, lambda ctx: (fu.usp_attention(
            ctx, qs[ctx.rank()], ks[ctx.rank()], vs[ctx.rank()], mesh, opts), ctx.traffic()))
        same = all(torch.equal(o, b[0]) for a, b in zip(res, loc.results) for o in a[0])
        traffic_ok = all(a[1][0] == 3 * b[1][0] and a[1][1] == 3 * b[1][1] for a, b in zip(res, loc.results))
        stats = [list(x[2]) for x in res]
        emit(check=f"peer_n{n}_r{r}_fp8{int(fp8)}", ok=bool(same and traffic_ok and all(st == [3, 0] for st in stats)),
             bit_identical_to_local=same, traffic_ok=traffic_ok, stats=stats)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which in ("all", "usp"):
        usp_cases()
    if which in ("all", "groups"):
        subgroups()
    if which in ("all", "dead"):
        dead_peer()
    if which in ("all", "peer"):
        peer_cases()

"""GPU: the bytes fastusp puts on the wire, compared byte for byte with the reference.

fusp_ctx_debug_wire keeps a device copy of every payload a rank sends.  The FP8 payloads are
held to the reference quantizer itself (oracle/_ref = uspsim's fp8.cpp:107-123 compiled here):
  * Ulysses-in slot t (protocols.cpp:139-153): [Q heads t*hp.. in the caller's dtype]
    [K codes of quantize(k_local).slice_heads(t*hp, hp)][V codes][k scale][v scale] --
    codes AND scale trailers memcmp-equal (per-block: one quantize per (b,h) slab);
  * ring hop 1 (protocols.cpp:113-121, 303-311): quantize(resharded chunk), where the chunk is
    the exact f32 decode(code)*scale values the Ulysses step produced; hop i > 1:
    quantize(dequantize(what the member received at hop i-1)) -- codes and scale equal.
The bf16 wire carries Q, K, V unchanged (the reference's f32 payloads at 2 bytes)."""
import numpy as np
import pytest
import torch

from oracle import ref, ref_available
from oracle import restate as R
from oracle.make_golden import qkv

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_ref():
    if not ref_available():
        pytest.skip("oracle/_ref not built")


def bf16_bytes(x):
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).bfloat16().view(torch.int16).numpy().view(np.uint8).ravel()


def quant(x, per_block):
    """reference quantize, per tensor or per (b,h) slab: (codes, scales[])."""
    if not per_block:
        c, s = ref.quantize(x)
        return c, np.array([s], np.float32)
    b, h = x.shape[:2]
    codes = np.empty(x.shape, np.uint8)
    scales = np.empty(b * h, np.float32)
    for i in range(b):
        for j in range(h):
            c, s = ref.quantize(x[i:i + 1, j:j + 1])
            codes[i, j] = c[0, 0]
            scales[i * h + j] = s
    return codes, scales


def dequant(codes, scales, per_block):
    if not per_block:
        return ref.dequantize(codes, float(scales[0]))
    b, h = codes.shape[:2]
    out = np.empty(codes.shape, np.float32)
    for i in range(b):
        for j in range(h):
            out[i, j] = ref.dequantize(codes[i:i + 1, j:j + 1], float(scales[i * h + j]))[0, 0]
    return out


def run(fu, n, r, fp8, per_block, b=1, h=8, sl=32):
    s = sl * n
    q, k, v = qkv((b, h, s, 128), (b, h, s, 128), seeds=(101, 102, 103))
    qs, ks, vs = (R.split_sequence(t, n) for t in (q, k, v))
    dev = [[torch.from_numpy(np.ascontiguousarray(x)).cuda().bfloat16() for x in t] for t in (qs, ks, vs)]
    mesh = fu.make_mesh(n, r)
    opts = fu.CommOptions(fp8_kv=fp8, fp8_block=int(per_block), pipelined_ring=True)

    def prog(ctx):
        ctx.debug_wire(True)
        fu.usp_attention(ctx, dev[0][ctx.rank()], dev[1][ctx.rank()], dev[2][ctx.rank()], mesh, opts)
        torch.cuda.current_stream().synchronize()
        return ctx.wire_records()

    return fu.run_protocol(n, prog).results, (qs, ks, vs)


@pytest.mark.parametrize("n,r", [(4, 2), (8, 4), (4, 4), (2, 1)])
@pytest.mark.parametrize("per_block", [False, True])
def test_fp8_wire_bytes_equal_reference_quantizer(cuda, fu, n, r, per_block):
    b, h, sl = (2 if per_block else 1), 8, 32
    recs, (qs, ks, vs) = run(fu, n, r, True, per_block, b=b, h=h, sl=sl)
    u = n // r
    hp = h // u
    blk = b * hp * sl * 128
    nsc = b * hp if per_block else 1
    slot_bytes = 2 * blk + 2 * blk + 8 * nsc
    slot_stride = (slot_bytes + 255) // 256 * 256
    # --- Ulysses-in slots (U > 1)
    for m in range(n):
        a2a = [x for x in recs[m] if x[0] == 0]
        if u == 1:
            assert not a2a
            continue
        (_, _, buf), = a2a
        kc, ksc = quant(ks[m], per_block)
        vc, vsc = quant(vs[m], per_block)
        for t in range(u):
            sl_ = slice(t * hp, (t + 1) * hp)
            slot = buf[t * slot_stride:t * slot_stride + slot_bytes]
            assert np.array_equal(slot[:2 * blk], bf16_bytes(qs[m][:, sl_]))
            assert np.array_equal(slot[2 * blk:3 * blk], kc[:, sl_].ravel())
            assert np.array_equal(slot[3 * blk:4 * blk], vc[:, sl_].ravel())
            tr = slot[4 * blk:].view(np.float32)
            if per_block:  # the slot's slabs (b, t*hp + hl) in [b][hl] order
                want_k = ksc.reshape(b, h)[:, sl_].ravel()
                want_v = vsc.reshape(b, h)[:, sl_].ravel()
            else:          # slice_heads keeps the tensor-wide scale (fp8.cpp:100-105)
                want_k, want_v = ksc, vsc
            assert np.array_equal(tr[:nsc], want_k) and np.array_equal(tr[nsc:], want_v)
    # --- ring hops
    if r == 1:
        return
    ug, rg = R.make_mesh(n, r)
    resh = {}
    for grp in ug:
        out = R.ulysses_input_reshard([qs[x] for x in grp], [ks[x] for x in grp], [vs[x] for x in grp],
                                      True, per_block)
        for pos, x in enumerate(grp):
            resh[x] = out[pos]
    C = b * hp * sl * u * 128
    for grp in rg:
        payload = {}  # (member, hop, part) -> (codes, scales)
        for hop in range(1, r):
            for p, m in enumerate(grp):
                for part in (1, 2):
                    if hop == 1:
                        src = resh[m][part]
                    else:
                        prev = grp[(p - 1) % r]
                        src = dequant(*payload[(prev, hop - 1, part)], per_block)
                    codes, scales = quant(src, per_block)
                    payload[(m, hop, part)] = (codes, scales)
                    (_, _, buf), = [x for x in recs[m] if x[0] == part and x[1] == hop]
                    assert np.array_equal(buf[:C], codes.ravel()), (m, hop, part)
                    assert np.array_equal(buf[C:].view(np.float32)[:len(scales)], scales), (m, hop, part)


def test_bf16_wire_carries_inputs_unchanged(cuda, fu):
    n, r, b, h, sl = 4, 2, 1, 8, 32
    recs, (qs, ks, vs) = run(fu, n, r, False, False, b=b, h=h, sl=sl)
    u, hp = n // r, h // (n // r)
    blk = b * hp * sl * 128
    slot_stride = (6 * blk + 255) // 256 * 256
    ug, rg = R.make_mesh(n, r)
    resh = {}
    for grp in ug:
        out = R.ulysses_input_reshard([qs[x] for x in grp], [ks[x] for x in grp], [vs[x] for x in grp], False)
        for pos, x in enumerate(grp):
            resh[x] = out[pos]
    for m in range(n):
        (_, _, buf), = [x for x in recs[m] if x[0] == 0]
        for t in range(u):
            sl_ = slice(t * hp, (t + 1) * hp)
            slot = buf[t * slot_stride:t * slot_stride + 6 * blk]
            want = np.concatenate([bf16_bytes(x[m][:, sl_]) for x in (qs, ks, vs)])
            assert np.array_equal(slot, want)
        for part in (1, 2):  # ring hop 1 forwards the resharded chunk as it arrived
            (_, _, buf), = [x for x in recs[m] if x[0] == part and x[1] == 1]
            assert np.array_equal(buf, bf16_bytes(resh[m][part]))

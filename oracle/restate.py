"""TEST INFRASTRUCTURE ONLY -- numpy restatement of the reference's hot path.

Each function restates one reference function (file:line under
/root/reference/proj).  Byte/integer work (the E4M3 codec, the quantizer, the
resharding data movement, the mesh) is bit-exact with the compiled reference
(pinned in tests/test_oracle.py against oracle/_ref and tests/golden).  The
floating-point attention is restated in float64, so it agrees with the
reference's float32 loop to ~1e-6, not bit-for-bit.

Never imported by the product package.
"""
from __future__ import annotations

import numpy as np

FP8_MAX = np.float32(448.0)      # fp8.hpp:15
FP8_MAX_CODE = 0x7E              # fp8.hpp:16
FP8_NAN_CODE = 0x7F              # fp8.hpp:17


# ---- rng.hpp:20-43 -----------------------------------------------------------
def rng_uniform(seed: int, n: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """uspsim::Rng(seed).uniform(lo,hi) x n  (rng.hpp:20-30).

    std::mt19937 seeded with uint32(seed ^ (seed >> 32)); numpy's legacy
    RandomState(int) uses the same init_genrand, so the raw streams agree.
    u = (next_u32() >> 8) * 2^-24 in float32, then lo + u*(hi-lo) in float32.
    """
    s32 = (seed ^ (seed >> 32)) & 0xFFFFFFFF
    bg = np.random.RandomState(s32)._bit_generator  # MT19937, init_genrand(s32)
    raw = bg.random_raw(n).astype(np.uint32)
    u = (raw >> np.uint32(8)).astype(np.float32) * np.float32(1.0 / 16777216.0)
    return (np.float32(lo) + u * (np.float32(hi) - np.float32(lo))).astype(np.float32)


def rng_tensor(seed: int, shape, lo=-1.0, hi=1.0) -> np.ndarray:
    return rng_uniform(seed, int(np.prod(shape)), lo, hi).reshape(shape)


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round float32 to the nearest bf16 value (RNE), returned as float32."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    lsb = (b >> np.uint32(16)) & np.uint32(1)
    r = (b + np.uint32(0x7FFF) + lsb) & np.uint32(0xFFFF0000)
    return r.view(np.float32)


# ---- fp8.cpp:18-68 ----------------------------------------------------------
def _magnitudes() -> np.ndarray:
    """magnitude_of(code) for codes 0x00..0x7E (fp8.cpp:18-35)."""
    vals = np.empty(127, np.float32)
    for c in range(127):
        e, m = (c >> 3) & 0xF, c & 7
        vals[c] = np.ldexp(np.float32(m), -9) if e == 0 else np.ldexp(np.float32(8 + m), e - 10)
    return vals


MAG = _magnitudes()


def decode_e4m3(codes) -> np.ndarray:
    """decode_e4m3 (fp8.cpp:39-43): NaN pattern -> NaN, else +-table[code&0x7F]."""
    c = np.asarray(codes, dtype=np.uint8)
    mag = np.concatenate([MAG, np.array([np.nan], np.float32)])[c & 0x7F]
    return np.where(c & 0x80, -mag, mag).astype(np.float32)


def encode_e4m3(x) -> np.ndarray:
    """encode_e4m3 (fp8.cpp:45-68): RNE, saturating to 0x7E, NaN -> 0x7F|sign."""
    x = np.asarray(x, dtype=np.float32)
    sign = np.where(np.signbit(x), 0x80, 0x00).astype(np.uint8)
    a = np.abs(x)
    isnan = np.isnan(x)
    a_safe = np.where(isnan, 0, a)
    # largest code whose value is <= a  (binary search at fp8.cpp:54-60)
    lo = np.clip(np.searchsorted(MAG, a_safe, side="right") - 1, 0, 126)
    below = MAG[lo]
    above = MAG[np.minimum(lo + 1, 126)]
    mid = np.float32(0.5) * (below + above)  # exact in f32 (fp8.cpp:64-65)
    code = np.where(a_safe < mid, lo, np.where(a_safe > mid, lo + 1, np.where(lo & 1, lo + 1, lo)))
    code = np.where(lo == 126, 126, code)
    code = np.where(a_safe >= FP8_MAX, FP8_MAX_CODE, code).astype(np.uint8)
    out = sign | code
    return np.where(isnan, sign | FP8_NAN_CODE, out).astype(np.uint8)


def quantize(x):
    """quantize (fp8.cpp:107-123): scale = max|x|/448 (1 if 0), codes = enc(x/scale)."""
    x = np.asarray(x, dtype=np.float32)
    if not np.all(np.isfinite(x)):
        i = int(np.flatnonzero(~np.isfinite(x.ravel()))[0])
        raise ValueError(f"quantize: non-finite element at flat index {i}")
    m = np.float32(np.max(np.abs(x))) if x.size else np.float32(0)
    scale = np.float32(m / FP8_MAX) if m > 0 else np.float32(1.0)
    return encode_e4m3(x / scale), scale


def dequantize(codes, scale) -> np.ndarray:
    """dequantize (fp8.cpp:125-130): decode(code) * scale in float32."""
    return (decode_e4m3(codes) * np.float32(scale)).astype(np.float32)


def fake_quant(x, per_block: bool = False) -> np.ndarray:
    """dequantize(quantize(x)); per_block quantizes every (b,h) slab on its own (the B200
    per-block option: uspsim::quantize applied to each slab's Tensor4 slice)."""
    x = np.asarray(x, np.float32)
    if not per_block:
        c, s = quantize(x)
        return dequantize(c, s)
    out = np.empty_like(x)
    for b in range(x.shape[0]):
        for h in range(x.shape[1]):
            c, s = quantize(x[b:b + 1, h:h + 1])
            out[b:b + 1, h:h + 1] = dequantize(c, s)
    return out


# ---- tensor.cpp:143-243 -----------------------------------------------------
def attention_with_lse(q, k, v):
    """attention_with_lse -> attention_core (tensor.cpp:143-202), in float64.

    logits z = (q.k) * (1/sqrt(D)); row max; w = exp(z - max); out = sum w v / sum w;
    lse = max + ln(sum w) (natural log).  Empty key set -> out 0, lse -inf (:161-164).
    """
    q, k, v = (np.asarray(t, dtype=np.float64) for t in (q, k, v))
    b, h, sq, d = q.shape
    if k.shape[2] == 0:
        return np.zeros(q.shape), np.full((b, h, sq), -np.inf)
    z = np.einsum("bhqd,bhkd->bhqk", q, k) * (1.0 / np.sqrt(d))
    m = z.max(axis=-1, keepdims=True)
    w = np.exp(z - m)
    den = w.sum(axis=-1, keepdims=True)
    out = np.einsum("bhqk,bhkd->bhqd", w, v) / den
    return out, (m + np.log(den))[..., 0]


def merge_lse(o1, l1, o2, l2):
    """merge_lse (tensor.cpp:204-243), float32, identity rows pass through untouched."""
    o1, o2 = np.asarray(o1, np.float32), np.asarray(o2, np.float32)
    l1, l2 = np.asarray(l1, np.float32), np.asarray(l2, np.float32)
    with np.errstate(invalid="ignore", over="ignore"):
        m = np.maximum(l1, l2)
        lse = (m + np.log(np.exp(l1 - m) + np.exp(l2 - m))).astype(np.float32)
        c1 = np.exp(l1 - lse).astype(np.float32)
        c2 = np.exp(l2 - lse).astype(np.float32)
        out = (c1[..., None] * o1 + c2[..., None] * o2).astype(np.float32)
    id2 = np.isneginf(l2)
    id1 = np.isneginf(l1) & ~id2
    out = np.where(id2[..., None], o1, np.where(id1[..., None], o2, out))
    lse = np.where(id2, l1, np.where(id1, l2, lse))
    return out, lse


# ---- mesh.cpp:34-79 ---------------------------------------------------------
class MeshError(ValueError):
    pass


def make_mesh(n: int, r: int):
    """make_mesh (mesh.cpp:34-55): rank = ring_idx*U + ulysses_idx."""
    if n < 1:
        raise MeshError(f"worker count must be >= 1, got {n}")
    if r < 1 or n % r:
        raise MeshError(f"ring dimension {r} does not divide worker count {n}")
    u = n // r
    ulysses = [[i * u + j for j in range(u)] for i in range(r)]
    ring = [[i * u + j for i in range(r)] for j in range(u)]
    return ulysses, ring


def build_mesh(n: int, max_ring: int, heads: int):
    """build_mesh (mesh.cpp:57-79): the LARGEST feasible R <= max_ring."""
    if n < 1:
        raise MeshError(f"worker count must be >= 1, got {n}")
    if max_ring < 1:
        raise MeshError(f"max_ring_dim_size must be >= 1, got {max_ring}")
    if heads < 1:
        raise MeshError(f"head count must be >= 1, got {heads}")
    for r in range(min(n, max_ring), 0, -1):
        if n % r == 0 and heads % (n // r) == 0:
            return r, n // r
    raise MeshError(f"no feasible (R,U) mesh for N={n}, max_ring_dim_size={max_ring}, H={heads}")


# ---- protocols.cpp ----------------------------------------------------------
def split_sequence(full, count: int):
    """split_sequence (protocols.cpp:10-21)."""
    s = full.shape[2]
    if s % count:
        raise ValueError(f"split_sequence: S={s} not divisible by shard count {count}")
    c = s // count
    return [full[:, :, i * c:(i + 1) * c] for i in range(count)]


def ulysses_input_reshard(qs, ks, vs, fp8: bool, per_block: bool = False):
    """detail::ulysses_input_reshard for one group (protocols.cpp:125-180).

    qs/ks/vs: the group members' local [B,H,S/N,D] shards in group order.
    With fp8, each member quantizes its WHOLE local K and V (:139-142, scale over
    all H heads), every destination -- including itself -- receives the
    dequantized head slice (:146-149, :163-179).  Q is never quantized.
    Returns per-member (q,k,v) [B,H/U,U*S/N,D] in group-position sequence order.
    """
    u = len(qs)
    h = qs[0].shape[1]
    if h % u:
        raise ValueError(f"ulysses: head count H={h} not divisible by ulysses dimension U={u}")
    hp = h // u
    if fp8:
        ks = [fake_quant(k, per_block) for k in ks]
        vs = [fake_quant(v, per_block) for v in vs]
    res = []
    for t in range(u):
        sl = slice(t * hp, (t + 1) * hp)
        res.append(tuple(np.concatenate([x[:, sl] for x in src], axis=2) for src in (qs, ks, vs)))
    return res


def ulysses_output_reshard(outs):
    """detail::ulysses_output_reshard (protocols.cpp:182-203): seq split -> head concat."""
    u = len(outs)
    s = outs[0].shape[2]
    if s % u:
        raise ValueError(f"ulysses: gathered sequence length S={s} not divisible by U={u}")
    sp = s // u
    return [np.concatenate([o[:, :, t * sp:(t + 1) * sp] for o in outs], axis=1) for t in range(u)]


def ring_attention(qs, ks, vs, fp8: bool, attn=attention_with_lse, per_block: bool = False):
    """ring_attention_serial == ring_attention_pipelined (protocols.cpp:237-319).

    Member p: acc = attn(q_p, k_p, v_p); round i=1..R-1 receives the chunk that
    originated at position (p-i) mod R and left-folds merge_lse (:265-266).
    With fp8 every hop re-quantizes the chunk it forwards from the dequantized
    values it holds (:113-121, :301-311); hop 1 quantizes the original chunk.
    """
    r = len(qs)
    res = []
    for p in range(r):
        o, l = attn(qs[p], ks[p], vs[p])
        o, l = np.asarray(o, np.float32), np.asarray(l, np.float32)
        for i in range(1, r):
            src = (p - i) % r
            kc, vc = ks[src], vs[src]
            if fp8:  # the chunk travelled i hops, re-quantized at each
                for _ in range(i):
                    kc, vc = fake_quant(kc, per_block), fake_quant(vc, per_block)
            po, pl = attn(qs[p], kc, vc)
            o, l = merge_lse(o, l, np.asarray(po, np.float32), np.asarray(pl, np.float32))
        res.append((o, l))
    return res


def usp_attention(q, k, v, n: int, r: int, fp8: bool = False, attn=attention_with_lse,
                  per_block: bool = False):
    """usp_attention (protocols.cpp:321-340) over all n ranks; returns the gathered output.

    Ulysses-in within each ulysses group, ring within each ring group, Ulysses-out.
    """
    u = n // r
    if q.shape[1] % u:
        raise ValueError(f"usp: head count H={q.shape[1]} not divisible by U={u}")
    qs, ks, vs = (split_sequence(np.asarray(t, np.float32), n) for t in (q, k, v))
    ug, rg = make_mesh(n, r)
    rs = {}
    for grp in ug:
        out = ulysses_input_reshard([qs[m] for m in grp], [ks[m] for m in grp],
                                    [vs[m] for m in grp], fp8, per_block)
        for pos, m in enumerate(grp):
            rs[m] = out[pos]
    red = {}
    for grp in rg:
        out = ring_attention([rs[m][0] for m in grp], [rs[m][1] for m in grp],
                             [rs[m][2] for m in grp], fp8, attn, per_block)
        for pos, m in enumerate(grp):
            red[m] = out[pos][0]
    final = {}
    for grp in ug:
        out = ulysses_output_reshard([red[m] for m in grp])
        for pos, m in enumerate(grp):
            final[m] = out[pos]
    return np.concatenate([final[i] for i in range(n)], axis=2)


# ---- producer prologue (NOT in the reference) ---------------------------
# The MMDiT block (FLUX) normalizes each Q/K head row with RMSNorm and applies
# rotary embedding before attention.  The reference's uspsim takes Q/K/V after that point,
# so there is no reference code to cite: this is the textbook definition the fused
# fusp_qk_prologue kernel is checked against, in float64.
def rms_norm(x, w, eps):
    x = np.asarray(x, np.float64)
    r = 1.0 / np.sqrt((x * x).mean(axis=-1, keepdims=True) + eps)
    return x * r * np.asarray(w, np.float64)


def rope_interleaved(x, cos, sin, pos0: int = 0):
    """Rotate pairs (x[2i], x[2i+1]) of every row at sequence position pos0 + s."""
    x = np.asarray(x, np.float64)
    s = x.shape[-2]
    c = np.asarray(cos, np.float64)[pos0:pos0 + s]
    n = np.asarray(sin, np.float64)[pos0:pos0 + s]
    x0, x1 = x[..., 0::2], x[..., 1::2]
    y = np.empty_like(x)
    y[..., 0::2] = x0 * c - x1 * n
    y[..., 1::2] = x0 * n + x1 * c
    return y


def qk_prologue(x, w=None, eps=1e-6, cos=None, sin=None, pos0: int = 0):
    y = np.asarray(x, np.float64)
    if w is not None:
        y = rms_norm(y, w, eps)
    if cos is not None:
        y = rope_interleaved(y, cos, sin, pos0)
    return y


def traffic_closed_form(b, h, s, d, n, r, fp8=False, w=4):
    """Per-rank bytes: all_to_all in+out, ring sends; self-slot free."""
    u = n // r
    hp, sl = h // u, s // n
    blk = b * hp * sl * d
    kv = (blk + 4) if fp8 else blk * w
    a2a = (u - 1) * (blk * w + 2 * kv) + (u - 1) * blk * w
    chunk = b * hp * (s // r) * d
    ring = (r - 1) * 2 * ((chunk + 4) if fp8 else chunk * w)
    return a2a, ring

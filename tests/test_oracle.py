"""CPU: pin the oracle before trusting it.

* the numpy restatement (oracle.restate) against the reference's own compiled
  library (oracle/_ref) and against the committed golden vectors (tests/golden);
* the SPEC.md known answers and the verified survey findings
  (D4 grid equivalence, D7 self-slot FP8 round trip, D10 build_mesh rule).
"""
import math

import numpy as np
import pytest

from oracle import ref, ref_available
from oracle import restate as R
from oracle.make_golden import ATTN_CASES, USP_CASES, fp8_grid, qkv

GOLD = __import__("os").path.join(__import__("os").path.dirname(__file__), "golden")
needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")


def gold(name):
    return np.load(f"{GOLD}/{name}.npz")


# ---- RNG (rng.hpp) -------------------------------------------------------------------------
@needs_ref
@pytest.mark.parametrize("seed", [0, 42, 2**32 + 5, 2**63 - 1])
def test_rng_stream_matches_reference(seed):
    assert np.array_equal(R.rng_uniform(seed, 5000, -3, 3), ref.rng_uniform(seed, 5000, -3, 3))


# ---- FP8 codec (fp8.cpp) --------------------------------------------------------------------
def test_fp8_constants_and_known_codes():
    # SPEC.md:100-102, 118-130
    assert R.decode_e4m3(np.array([0x7E], np.uint8))[0] == 448.0
    assert R.decode_e4m3(np.array([0x01], np.uint8))[0] == 2.0**-9
    assert np.isnan(R.decode_e4m3(np.array([0x7F, 0xFF], np.uint8))).all()
    assert R.encode_e4m3(np.array([0.0]))[0] == 0x00
    assert R.encode_e4m3(np.array([1000.0]))[0] == 0x7E
    assert R.encode_e4m3(np.array([-1000.0]))[0] == 0xFE
    d = R.decode_e4m3(np.array([0x80], np.uint8))[0]
    assert d == 0 and math.copysign(1, d) < 0
    # exhaustive round trip over all non-NaN codes, sign symmetry
    codes = np.array([c for c in range(256) if (c & 0x7F) != 0x7F], np.uint8)
    assert np.array_equal(R.encode_e4m3(R.decode_e4m3(codes)), codes)
    mags = R.decode_e4m3(np.arange(0x7F, dtype=np.uint8))
    assert np.all(np.diff(mags) > 0)


def test_fp8_encode_golden():
    g = gold("fp8")
    assert np.array_equal(R.encode_e4m3(fp8_grid()), g["enc_codes"])
    assert np.array_equal(R.decode_e4m3(g["dec_codes"]), g["dec_vals"], equal_nan=True)


def test_quantize_golden_and_spec():
    g = gold("fp8")
    c, s = R.quantize(g["q_spec_x"])
    assert list(c.ravel()) == [0x7E, 0xF6, 0x00] and s == 1.0
    c, s = R.quantize(g["q_zeros_x"])
    assert s == 1.0 and not c.any()
    for name, t in (("u1", R.rng_tensor(11, (1, 4, 16, 128))),
                    ("u3", R.rng_tensor(12, (2, 3, 40, 128), -3, 3))):
        c, s = R.quantize(t)
        assert np.array_equal(c, g[f"q_{name}_codes"]) and s == g[f"q_{name}_scale"][0]


def test_quantize_gaussian_rms():
    # 4096 Box-Muller normals over Rng(123), RMS relative error <= 3%
    u = R.rng_uniform(123, 4096, 0, 1).astype(np.float64)
    u1, u2 = np.maximum(u[0::2], 1e-12), u[1::2]
    z = np.concatenate([np.sqrt(-2 * np.log(u1)) * np.cos(2 * np.pi * u2),
                        np.sqrt(-2 * np.log(u1)) * np.sin(2 * np.pi * u2)]).astype(np.float32)
    x = R.dequantize(*R.quantize(z))
    assert np.sqrt(np.mean((x - z) ** 2)) / np.sqrt(np.mean(z**2)) <= 0.03


def test_quantize_rejects_non_finite():
    with pytest.raises(ValueError, match="non-finite element at flat index 2"):
        R.quantize(np.array([1.0, 2.0, np.nan], np.float32))


@needs_ref
def test_encode_matches_reference_random():
    x = np.random.RandomState(1).standard_normal(100000).astype(np.float32) * 200
    assert np.array_equal(R.encode_e4m3(x), ref.encode_e4m3(x))


@needs_ref
def test_quantize_matches_reference_errors():
    with pytest.raises(Exception) as e:
        ref.quantize(np.array([0, np.inf, 0, 0], np.float32).reshape(1, 1, 1, 4))
    assert e.value.kind == "invalid_argument" and "flat index 1" in e.value.msg


# ---- attention + merge (tensor.cpp) -------------------------------------------------------------
@pytest.mark.parametrize("name,b,h,sq,skv", ATTN_CASES)
def test_attention_restatement_vs_golden(name, b, h, sq, skv):
    g = gold("attention")
    q, k, v = qkv((b, h, sq, 128), (b, h, skv, 128))
    o, l = R.attention_with_lse(q, k, v)
    assert np.abs(o - g[f"{name}_out"]).max() < 2e-6
    assert np.abs(l - g[f"{name}_lse"]).max() < 2e-6


def test_attention_spec_examples():
    # S=1 -> the single V row; identical keys -> mean of V
    q = np.array([[[[0.3, -1.0]]]]); k = np.array([[[[2.0, 1.0]]]]); v = np.array([[[[5.0, -7.0]]]])
    o, l = R.attention_with_lse(q, k, v)
    assert np.allclose(o, v)
    k2 = np.ones((1, 1, 2, 1)); v2 = np.array([[[[2.0], [4.0]]]])
    o, l = R.attention_with_lse(np.ones((1, 1, 3, 1)), k2, v2)
    assert np.allclose(o, 3.0)
    # lse: single key with zero logit -> 0; two equal logits z -> z + ln 2
    _, l = R.attention_with_lse(np.zeros((1, 1, 1, 4)), np.ones((1, 1, 1, 4)), np.ones((1, 1, 1, 4)))
    assert abs(l[0, 0, 0]) < 1e-12
    _, l = R.attention_with_lse(np.ones((1, 1, 1, 4)), np.ones((1, 1, 2, 4)), np.ones((1, 1, 2, 4)))
    assert abs(l[0, 0, 0] - (2.0 + math.log(2))) < 1e-12


def test_merge_identity_and_golden():
    g = gold("attention")
    o, l = R.merge_lse(g["merge_o1"], g["merge_l1"], g["merge_o2"], g["merge_l2"])
    assert np.abs(o - g["merge_out"]).max() < 1e-6 and np.abs(l - g["merge_lse"]).max() < 1e-6
    # identity element (tensor.cpp:223-232) is bit-exact on both sides
    ident_l = np.full_like(g["merge_l1"], -np.inf)
    o, l = R.merge_lse(g["merge_o1"], g["merge_l1"], np.zeros_like(g["merge_o1"]), ident_l)
    assert np.array_equal(o, g["merge_o1"]) and np.array_equal(l, g["merge_l1"])
    o, l = R.merge_lse(np.zeros_like(g["merge_o1"]), ident_l, g["merge_o1"], g["merge_l1"])
    assert np.array_equal(o, g["merge_o1"])
    # merge(x, x) -> lse + ln 2, O unchanged
    o, l = R.merge_lse(g["merge_o1"], g["merge_l1"], g["merge_o1"], g["merge_l1"])
    assert np.abs(l - (g["merge_l1"] + np.float32(math.log(2)))).max() < 1e-5
    assert np.abs(o - g["merge_o1"]).max() < 1e-6


@needs_ref
def test_merge_matches_reference():
    q, k, v = qkv((1, 3, 20, 128), (1, 3, 70, 128))
    a = ref.attention_with_lse(q, k[:, :, :30], v[:, :, :30])
    b = ref.attention_with_lse(q, k[:, :, 30:], v[:, :, 30:])
    ro, rl = ref.merge_lse(*a, *b)
    o, l = R.merge_lse(*a, *b)
    assert np.abs(o - ro).max() < 1e-6 and np.abs(l - rl).max() < 1e-6


# ---- mesh (mesh.cpp) -----------------------------------------------------------------------------
def test_build_mesh_largest_feasible_r():
    # the code picks the LARGEST feasible R (mesh.cpp:63-67)
    assert R.build_mesh(8, 2, 24) == (2, 4)
    assert R.build_mesh(4, 2, 8) == (2, 2)
    assert R.build_mesh(8, 4, 24) == (4, 2)
    assert R.build_mesh(8, 8, 24) == (8, 1)
    with pytest.raises(R.MeshError):
        R.build_mesh(4, 1, 3)
    ug, rg = R.make_mesh(4, 2)
    assert ug == [[0, 1], [2, 3]] and rg == [[0, 2], [1, 3]]


@needs_ref
@pytest.mark.parametrize("n", [1, 2, 3, 4, 6, 8])
@pytest.mark.parametrize("max_ring", [1, 2, 4, 8])
@pytest.mark.parametrize("heads", [1, 3, 8, 24])
def test_build_mesh_matches_reference(n, max_ring, heads):
    try:
        want = ref.build_mesh(n, max_ring, heads)
    except Exception as e:  # noqa: BLE001
        assert e.kind == "MeshError"
        with pytest.raises(R.MeshError):
            R.build_mesh(n, max_ring, heads)
        return
    assert R.build_mesh(n, max_ring, heads) == want
    ug, rg = ref.make_mesh(n, want[0])
    mu, mr = R.make_mesh(n, want[0])
    assert ug.tolist() == mu and rg.tolist() == mr


# ---- protocols (protocols.cpp) -------------------------------------------------------------------
@pytest.mark.parametrize("n,r,fp8,h,s", USP_CASES)
def test_usp_restatement_vs_golden(n, r, fp8, h, s):
    g = gold("usp")
    q, k, v = qkv((1, h, s, 128), (1, h, s, 128))
    key = f"n{n}_r{r}_{'fp8' if fp8 else 'f32'}"
    o = R.usp_attention(q, k, v, n, r, fp8=fp8)
    assert np.abs(o - g[key + "_out"]).max() < 5e-6
    # traffic closed forms, reference wire width w = 4 (f32)
    a2a, ring = R.traffic_closed_form(1, h, s, 128, n, r, fp8=fp8, w=4)
    assert np.all(g[key + "_a2a"] == a2a) and np.all(g[key + "_send"] == ring)


def test_usp_equals_full_attention():
    # D4: every (N, R) composition equals the full-sequence oracle
    q, k, v = qkv((1, 8, 32, 128), (1, 8, 32, 128))
    full, _ = R.attention_with_lse(q, k, v)
    for n, r in ((2, 1), (2, 2), (4, 2), (8, 4)):
        assert np.abs(R.usp_attention(q, k, v, n, r) - full).max() < 5e-6


@needs_ref
def test_fp8_selfslot_roundtrip_and_q_untouched():
    # D7: the Ulysses self slot is quantized too; Q is never quantized
    q, k, v = qkv((1, 4, 16, 128), (1, 4, 16, 128))
    rq, rk, rv = ref.ulysses_input_reshard(q, k, v, 2, fp8=True)
    ks = R.split_sequence(k, 2)
    want = R.ulysses_input_reshard(R.split_sequence(q, 2), ks, R.split_sequence(v, 2), True)
    for r in range(2):
        assert np.array_equal(rq[r], want[r][0])
        assert np.array_equal(rk[r], want[r][1])
        assert np.array_equal(rv[r], want[r][2])
    assert np.array_equal(rk[0][:, :, :8], R.fake_quant(ks[0])[:, :2])


@needs_ref
@pytest.mark.parametrize("n", [2, 4])
@pytest.mark.parametrize("fp8", [False, True])
def test_ring_pipelined_equals_serial_reference(n, fp8):
    q, k, v = qkv((1, 2, 16 * n, 128), (1, 2, 16 * n, 128))
    a = ref.ring_attention(q, k, v, n, fp8=fp8, pipelined=False)
    b = ref.ring_attention(q, k, v, n, fp8=fp8, pipelined=True)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@needs_ref
def test_reference_error_classes():
    q = np.zeros((1, 3, 4, 8), np.float32)
    with pytest.raises(Exception) as e:
        ref.usp_attention(q, q, q, 2, 1)           # H=3 not divisible by U=2
    assert e.value.kind == "ShapeError" and "H=3" in e.value.msg
    bad = q.copy(); bad[0, 0, 0, 0] = np.nan
    with pytest.raises(Exception) as e:
        ref.usp_attention(bad, q, q, 1, 1)
    assert e.value.kind == "invalid_argument" and "non-finite" in e.value.msg


def test_qk_prologue_restatement_properties():
    """The prologue oracle (not in the reference): RMSNorm gives unit mean square with unit
    weights; RoPE is an isometry on each pair and makes q.k depend only on the position gap."""
    x = R.rng_tensor(3, (1, 2, 16, 128), -3, 3).astype(np.float64)
    y = R.rms_norm(x, np.ones(128), 0.0)
    assert np.allclose((y * y).mean(-1), 1.0, atol=1e-12)
    inv = 10000.0 ** (-np.arange(0, 128, 2) / 128)
    ang = np.arange(64)[:, None] * inv[None, :]
    cos, sin = np.cos(ang), np.sin(ang)
    z = R.rope_interleaved(x, cos, sin)
    pair = lambda t: t[..., 0::2] ** 2 + t[..., 1::2] ** 2
    assert np.allclose(pair(z), pair(x), rtol=1e-12)
    assert np.array_equal(R.rope_interleaved(x, np.ones((16, 64)), np.zeros((16, 64))), x)
    q, k = x[0, 0, :1], x[0, 1, :1]
    d1 = R.rope_interleaved(q, cos, sin, 5) @ R.rope_interleaved(k, cos, sin, 2).T
    d2 = R.rope_interleaved(q, cos, sin, 40) @ R.rope_interleaved(k, cos, sin, 37).T
    assert np.allclose(d1, d2, rtol=1e-10)
    assert np.array_equal(R.qk_prologue(x), x)

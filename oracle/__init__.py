"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the USP attention hot path.

Two oracles live here, and nothing in the product (``paper_2602_10940_b200``)
may import either of them; only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` use them, and only
as the checker or as the timed CPU baseline:

* ``oracle.ref`` -- ctypes handle on ``oracle/_ref/libuspsim_ref.so``, the
  reference's *own* C++ library compiled from ``/root/reference/proj/src`` by
  ``oracle/Makefile`` (two one-line compile fixes applied by declaration, see
  ``oracle/shim``).  This is the ground truth.
* ``oracle.restate`` -- a numpy restatement of the same algorithms, each
  function citing the reference file:line it follows.  It is pinned against
  ``oracle.ref`` and against ``tests/golden`` in the CPU test suite and is what
  the GPU box falls back to for large randomized cases.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libuspsim_ref.so")
REF_SRC = "/root/reference/proj"

ERR_NAMES = {1: "ShapeError", 2: "MeshError", 3: "FabricError", 4: "invalid_argument",
             5: "DeadlockError", 6: "WorkerFailure", 9: "error"}


class RefError(RuntimeError):
    """An exception thrown by the reference library; ``kind`` names its class."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERR_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERR_NAMES.get(code, "error")
        self.msg = msg


def build_ref(force: bool = False) -> bool:
    """Compile oracle/_ref from the reference sources (only where they exist)."""
    if os.path.exists(REF_SO) and not force:
        return True
    if not os.path.isdir(REF_SRC):
        return False
    subprocess.run(["make", "-s", "-C", HERE, "-j8"], check=True)
    return os.path.exists(REF_SO)


_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(REF_SO):
            build_ref()
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} not built (run `make -C oracle`)")
        lib = ctypes.CDLL(REF_SO)
        lib.ref_last_error.restype = ctypes.c_char_p
        _lib = lib
    return _lib


def ref_available() -> bool:
    try:
        _load()
        return True
    except (FileNotFoundError, OSError):
        return False


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _chk(code: int):
    if code != 0:
        raise RefError(code, _load().ref_last_error().decode())


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


I64 = ctypes.c_int64


class ref:  # noqa: N801 -- namespace mirroring uspsim::
    """ctypes wrappers over oracle/_ref (the reference's compiled code)."""

    @staticmethod
    def encode_e4m3(x) -> np.ndarray:
        x = _f32(x)
        out = np.empty(x.shape, np.uint8)
        _chk(_load().ref_encode_e4m3(_p(x), _p(out), I64(x.size)))
        return out

    @staticmethod
    def decode_e4m3(c) -> np.ndarray:
        c = np.ascontiguousarray(c, dtype=np.uint8)
        out = np.empty(c.shape, np.float32)
        _chk(_load().ref_decode_e4m3(_p(c), _p(out), I64(c.size)))
        return out

    @staticmethod
    def quantize(x):
        x = _f32(x)
        b, h, s, d = x.shape
        codes = np.empty(x.shape, np.uint8)
        scale = np.zeros(1, np.float32)
        _chk(_load().ref_quantize(_p(x), I64(b), I64(h), I64(s), I64(d), _p(codes), _p(scale)))
        return codes, np.float32(scale[0])

    @staticmethod
    def dequantize(codes, scale):
        codes = np.ascontiguousarray(codes, dtype=np.uint8)
        b, h, s, d = codes.shape
        out = np.empty(codes.shape, np.float32)
        _chk(_load().ref_dequantize(_p(codes), ctypes.c_float(scale), I64(b), I64(h), I64(s),
                                    I64(d), _p(out)))
        return out

    @staticmethod
    def attention_with_lse(q, k, v, f64: bool = False):
        dt = np.float64 if f64 else np.float32
        q, k, v = (np.ascontiguousarray(t, dtype=dt) for t in (q, k, v))
        b, h, sq, d = q.shape
        skv = k.shape[2]
        out = np.empty(q.shape, dt)
        lse = np.empty((b, h, sq), dt)
        fn = _load().ref_attention_with_lse_f64 if f64 else _load().ref_attention_with_lse_f32
        _chk(fn(_p(q), _p(k), _p(v), I64(b), I64(h), I64(sq), I64(skv), I64(d), _p(out), _p(lse)))
        return out, lse

    @staticmethod
    def attention_reference(q, k, v):
        q, k, v = _f32(q), _f32(k), _f32(v)
        b, h, sq, d = q.shape
        out = np.empty(q.shape, np.float32)
        _chk(_load().ref_attention_reference_f32(_p(q), _p(k), _p(v), I64(b), I64(h), I64(sq),
                                                 I64(k.shape[2]), I64(d), _p(out)))
        return out

    @staticmethod
    def merge_lse(o1, l1, o2, l2):
        o1, l1, o2, l2 = _f32(o1), _f32(l1), _f32(o2), _f32(l2)
        b, h, s, d = o1.shape
        out = np.empty(o1.shape, np.float32)
        lse = np.empty((b, h, s), np.float32)
        _chk(_load().ref_merge_lse_f32(_p(o1), _p(l1), _p(o2), _p(l2), I64(b), I64(h), I64(s),
                                       I64(d), _p(out), _p(lse)))
        return out, lse

    @staticmethod
    def build_mesh(n, max_ring, heads):
        r, u = ctypes.c_int(), ctypes.c_int()
        _chk(_load().ref_build_mesh(n, max_ring, heads, ctypes.byref(r), ctypes.byref(u)))
        return r.value, u.value

    @staticmethod
    def make_mesh(n, r):
        ug = np.zeros(n, np.int32)
        rg = np.zeros(n, np.int32)
        _chk(_load().ref_make_mesh(n, r, _p(ug), _p(rg)))
        return ug.reshape(r, n // r), rg.reshape(n // r, r)

    @staticmethod
    def rng_uniform(seed: int, n: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
        out = np.empty(n, np.float32)
        _chk(_load().ref_rng_uniform(ctypes.c_uint64(seed), I64(n), ctypes.c_float(lo),
                                     ctypes.c_float(hi), _p(out)))
        return out

    @staticmethod
    def usp_attention(q, k, v, n, r, fp8=False, pipelined=False, traffic=False):
        q, k, v = _f32(q), _f32(k), _f32(v)
        b, h, s, d = q.shape
        out = np.empty(q.shape, np.float32)
        a2a = np.zeros(n, np.uint64)
        snd = np.zeros(n, np.uint64)
        _chk(_load().ref_usp_attention(n, r, int(fp8), int(pipelined), _p(q), _p(k), _p(v), I64(b),
                                       I64(h), I64(s), I64(d), _p(out), _p(a2a), _p(snd)))
        return (out, a2a, snd) if traffic else out

    @staticmethod
    def usp_report(q, k, v, n, r, fp8=False, pipelined=False):
        """(TrafficLog JSON, Timeline JSON) of the reference's usp_attention run."""
        import json
        q, k, v = _f32(q), _f32(k), _f32(v)
        b, h, s, d = q.shape
        tb = ctypes.create_string_buffer(1 << 20)
        lb = ctypes.create_string_buffer(1 << 20)
        _chk(_load().ref_usp_report(n, r, int(fp8), int(pipelined), _p(q), _p(k), _p(v), I64(b),
                                    I64(h), I64(s), I64(d), tb, ctypes.c_size_t(1 << 20), lb,
                                    ctypes.c_size_t(1 << 20)))
        return json.loads(tb.value.decode()), json.loads(lb.value.decode())

    @staticmethod
    def ulysses_attention(q, k, v, n, fp8=False):
        q, k, v = _f32(q), _f32(k), _f32(v)
        b, h, s, d = q.shape
        out = np.empty(q.shape, np.float32)
        _chk(_load().ref_ulysses_attention(n, int(fp8), _p(q), _p(k), _p(v), I64(b), I64(h),
                                           I64(s), I64(d), _p(out)))
        return out

    @staticmethod
    def ring_attention(q, k, v, n, fp8=False, pipelined=False):
        q, k, v = _f32(q), _f32(k), _f32(v)
        b, h, s, d = q.shape
        out = np.empty(q.shape, np.float32)
        lse = np.empty((b, h, s), np.float32)
        _chk(_load().ref_ring_attention(n, int(fp8), int(pipelined), _p(q), _p(k), _p(v), I64(b),
                                        I64(h), I64(s), I64(d), _p(out), _p(lse)))
        return out, lse

    @staticmethod
    def ulysses_input_reshard(q, k, v, n, fp8=False):
        q, k, v = _f32(q), _f32(k), _f32(v)
        b, h, s, d = q.shape
        shp = (n, b, h // n, s, d)
        rq, rk, rv = (np.empty(shp, np.float32) for _ in range(3))
        _chk(_load().ref_ulysses_input_reshard(n, int(fp8), _p(q), _p(k), _p(v), I64(b), I64(h),
                                               I64(s), I64(d), _p(rq), _p(rk), _p(rv)))
        return rq, rk, rv

    @staticmethod
    def time_attention(nthreads, sq, skv, d, seed=42):
        sec = ctypes.c_double()
        chk = ctypes.c_float()
        _chk(_load().ref_time_attention(nthreads, I64(sq), I64(skv), I64(d), ctypes.c_uint64(seed),
                                        ctypes.byref(sec), ctypes.byref(chk)))
        return sec.value, chk.value

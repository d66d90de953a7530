"""ctypes binding of libfastusp.so (the C ABI declared in include/fastusp.h).

The product path is the in-tree shared library; there is no CPU or PyTorch
fallback.  If the library is missing this module raises on first use.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "lib", "libfastusp.so")
# Kernel-variant experiments (tools/build_variants.sh) load an in-tree variant build instead.
if os.environ.get("FUSP_VARIANT"):
    LIB_PATH = os.path.join(PKG, "variants", os.environ["FUSP_VARIANT"], "libfastusp.so")

F32, F16, BF16, E4M3 = 0, 1, 2, 3

STATUS_NAMES = {0: "OK", 1: "ShapeError", 2: "MeshError", 3: "FabricError", 4: "invalid_argument",
                5: "DeadlockError", 10: "CudaError", 11: "NcclError", 12: "OutOfMemory",
                13: "Unsupported"}


class FuspError(RuntimeError):
    """Raised for a non-OK fusp_status; ``kind`` is the reference exception class name."""

    def __init__(self, code: int, msg: str):
        self.code = code
        self.kind = STATUS_NAMES.get(code, f"status{code}")
        self.msg = msg
        super().__init__(f"{self.kind}: {msg}")


class ShapeError(FuspError):
    pass


class MeshError(FuspError):
    pass


class FabricError(FuspError):
    pass


class InvalidArgument(FuspError, ValueError):
    pass


class DeadlockError(FuspError):
    """= uspsim::DeadlockError (fabric.hpp:112-116): a stalled or failed peer."""


_EXC = {1: ShapeError, 2: MeshError, 3: FabricError, 4: InvalidArgument, 5: DeadlockError}


class Shape4(ctypes.Structure):
    _fields_ = [("b", ctypes.c_int64), ("h", ctypes.c_int64), ("s", ctypes.c_int64),
                ("d", ctypes.c_int64)]


class CommOptions(ctypes.Structure):
    _fields_ = [("fp8_kv", ctypes.c_int), ("pipelined_ring", ctypes.c_int),
                ("out_dtype", ctypes.c_int), ("check_finite", ctypes.c_int),
                ("fp8_block", ctypes.c_int)]


class QKPrologue(ctypes.Structure):
    _fields_ = [("q_norm_weight", ctypes.c_void_p), ("k_norm_weight", ctypes.c_void_p),
                ("eps", ctypes.c_float), ("rope_cos", ctypes.c_void_p),
                ("rope_sin", ctypes.c_void_p), ("rope_rows", ctypes.c_int64),
                ("rope_pos0", ctypes.c_int64)]


def build(force: bool = False) -> str:
    """Compile libfastusp.so in-tree with nvcc for sm_100a (Makefile in this package)."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-s", "-C", PKG, "-j8"], check=True)
    return LIB_PATH


_lib = None

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_SIGS = {
    "fusp_last_error": (ctypes.c_char_p, []),
    "fusp_version": (ctypes.c_char_p, []),
    "fusp_kernel_launch_count": (ctypes.c_uint64, []),
    "fusp_attention_schedule": (ctypes.c_int, [ctypes.c_int, ctypes.c_int]),
    "fusp_attention_trace": (ctypes.c_int, [ctypes.c_int, _P, ctypes.c_size_t]),
    "fusp_encode_e4m3": (ctypes.c_int, [_P, _I64, _P, _P]),
    "fusp_decode_e4m3": (ctypes.c_int, [_P, _I64, _P, _P]),
    "fusp_quantize_e4m3": (ctypes.c_int, [_P, ctypes.c_int, _I64, _P, _P, ctypes.c_int, _P]),
    "fusp_dequantize_e4m3": (ctypes.c_int, [_P, _P, _I64, _P, ctypes.c_int, _P]),
    "fusp_requantize_e4m3": (ctypes.c_int, [_P, _P, _I64, _I64, _P, _P, _P]),
    "fusp_quantize_e4m3_blocks": (ctypes.c_int, [_P, ctypes.c_int, _I64, _I64, _P, _P, _P]),
    "fusp_dequantize_e4m3_blocks": (ctypes.c_int, [_P, _P, _I64, _I64, _P, ctypes.c_int, _P]),
    "fusp_attention_with_lse": (ctypes.c_int, [_P, _P, _P, ctypes.c_int, Shape4, _I64, _P,
                                               ctypes.c_int, _P, _P]),
    "fusp_attention_with_lse_ex": (ctypes.c_int, [_P, _P, _P, ctypes.c_int, ctypes.c_int, Shape4,
                                                  _I64, _P, ctypes.c_int, _P, _P]),
    "fusp_stage_f16": (ctypes.c_int, [_P, ctypes.c_int, _I64, _I64, _P, _P, _P]),
    "fusp_merge_lse": (ctypes.c_int, [_P, _P, _P, _P, Shape4, _P, _P, _P]),
    "fusp_mesh_build": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, _P, _P]),
    "fusp_mesh_make": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _P, _P]),
    "fusp_fabric_create": (ctypes.c_int, [ctypes.c_int, _P]),
    "fusp_fabric_destroy": (ctypes.c_int, [_P]),
    "fusp_ctx_create_local": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, _P]),
    "fusp_nccl_unique_id": (ctypes.c_int, [_P]),
    "fusp_ctx_create_nccl": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P]),
    "fusp_ctx_destroy": (ctypes.c_int, [_P]),
    "fusp_ctx_rank": (ctypes.c_int, [_P]),
    "fusp_ctx_world": (ctypes.c_int, [_P]),
    "fusp_ctx_traffic": (ctypes.c_int, [_P, _P, _P]),
    "fusp_ctx_reset_traffic": (ctypes.c_int, [_P]),
    "fusp_ctx_traffic_json": (ctypes.c_int, [_P, _P, ctypes.c_size_t, _P]),
    "fusp_ctx_timeline_json": (ctypes.c_int, [_P, _P, ctypes.c_size_t, _P]),
    "fusp_ctx_ring_timings": (ctypes.c_int, [_P, ctypes.c_int, _P, _P, _P]),
    "fusp_usp_attention": (ctypes.c_int, [_P, ctypes.c_int, _P, _P, _P, ctypes.c_int, Shape4, _P,
                                          ctypes.POINTER(CommOptions), _P]),
    "fusp_usp_attention_ex": (ctypes.c_int, [_P, ctypes.c_int, _P, _P, _P, ctypes.c_int, Shape4,
                                             _P, ctypes.POINTER(CommOptions),
                                             ctypes.POINTER(QKPrologue), _P]),
    "fusp_usp_attention_proj": (ctypes.c_int, [_P, ctypes.c_int, _P, _P, _P, ctypes.c_int, Shape4,
                                               _P, ctypes.POINTER(CommOptions),
                                               ctypes.POINTER(QKPrologue), _P, _I64, _P,
                                               ctypes.c_int, _P]),
    "fusp_out_projection": (ctypes.c_int, [_P, ctypes.c_int, Shape4, _P, _I64, _P, ctypes.c_int, _P]),
    "fusp_usp_block": (ctypes.c_int, [_P, ctypes.c_int, _P, ctypes.c_int, _I64, _I64, _I64, _P,
                                      ctypes.c_int, ctypes.POINTER(QKPrologue), _P, _I64, _P,
                                      ctypes.c_int, ctypes.POINTER(CommOptions), _P]),
    "fusp_ulysses_attention": (ctypes.c_int, [_P, _P, _P, _P, ctypes.c_int, Shape4, _P,
                                              ctypes.POINTER(CommOptions), _P]),
    "fusp_ring_attention": (ctypes.c_int, [_P, _P, _P, _P, ctypes.c_int, Shape4, _P, _P,
                                           ctypes.POINTER(CommOptions), _P]),
    "fusp_usp_attention_host": (ctypes.c_int, [_P, ctypes.c_int, _P, _P, _P, ctypes.c_int, Shape4,
                                               _P, ctypes.POINTER(CommOptions), _P]),
    "fusp_usp_attention_lse": (ctypes.c_int, [_P, ctypes.c_int, _P, _P, _P, ctypes.c_int, Shape4,
                                              _P, _P, ctypes.POINTER(CommOptions), _P]),
    "fusp_ctx_debug_wire": (ctypes.c_int, [_P, ctypes.c_int]),
    "fusp_ctx_debug_wire_count": (ctypes.c_int, [_P]),
    "fusp_ctx_debug_wire_get": (ctypes.c_int, [_P, ctypes.c_int, _P, _P, _P, ctypes.c_size_t, _P]),
    "fusp_ctx_synchronize": (ctypes.c_int, [_P, _P, ctypes.c_double]),
    "fusp_group_create": (ctypes.c_int, [_P, _P, ctypes.c_int, _P]),
    "fusp_group_destroy": (ctypes.c_int, [_P]),
    "fusp_group_size": (ctypes.c_int, [_P]),
    "fusp_group_position": (ctypes.c_int, [_P]),
    "fusp_ulysses_attention_group": (ctypes.c_int, [_P, _P, _P, _P, _P, ctypes.c_int, Shape4, _P,
                                                    _P, ctypes.POINTER(CommOptions), _P]),
    "fusp_ring_attention_group": (ctypes.c_int, [_P, _P, _P, _P, _P, ctypes.c_int, Shape4, _P, _P,
                                                 ctypes.POINTER(CommOptions), _P]),
    "fusp_ulysses_input_reshard": (ctypes.c_int, [_P, _P, _P, _P, _P, ctypes.c_int, Shape4, _P, _P,
                                                  _P, ctypes.c_int, ctypes.POINTER(CommOptions),
                                                  _P]),
    "fusp_ulysses_output_reshard": (ctypes.c_int, [_P, _P, _P, ctypes.c_int, Shape4, _P, _P]),
    "fusp_graph_capture_usp": (ctypes.c_int, [_P, ctypes.c_int, _P, _P, _P, ctypes.c_int, Shape4,
                                              _P, ctypes.POINTER(CommOptions), ctypes.c_int, _I64,
                                              _I64, _P, _P]),
    "fusp_graph_capture_block": (ctypes.c_int, [_P, ctypes.c_int, _P, ctypes.c_int, _I64, _I64, _I64,
                                                _P, ctypes.c_int, ctypes.POINTER(QKPrologue), _P,
                                                _I64, _P, ctypes.c_int, ctypes.POINTER(CommOptions),
                                                ctypes.c_int, _I64, _I64, _P, _P]),
    "fusp_ctx_peer_enable": (ctypes.c_int, [_P, ctypes.c_size_t]),
    "fusp_ctx_peer_window": (ctypes.c_int, [_P, ctypes.c_size_t, _P]),
    "fusp_ctx_peer_open": (ctypes.c_int, [_P, _P]),
    "fusp_peer_window_bytes": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, Shape4,
                                              ctypes.POINTER(CommOptions), _P]),
    "fusp_ctx_peer_stats": (ctypes.c_int, [_P, _P, _P]),
    "fusp_ctx_peer_disable": (ctypes.c_int, [_P]),
    "fusp_graph_launch": (ctypes.c_int, [_P, _P]),
    "fusp_graph_destroy": (ctypes.c_int, [_P]),
}

EXPORTED = tuple(_SIGS)


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(
                f"{LIB_PATH} is not built; run `make -C {PKG}` (or __graft_entry__.build()). "
                "fastusp has no CPU fallback.")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name, None)
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(code: int) -> None:
    if code != 0:
        msg = lib().fusp_last_error().decode()
        raise _EXC.get(code, FuspError)(code, msg)

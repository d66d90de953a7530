"""Python host mirror of the reference uspsim API, over the fastusp C ABI.

Names, argument meanings and error classes follow the reference
(/root/reference/proj/include/uspsim/{tensor,fp8,mesh,protocols}.hpp); tensors
are torch CUDA tensors (device memory plumbing only -- every computation runs in
libfastusp.so's sm_100a kernels).
"""
from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import torch

from . import _lib
from ._lib import (BF16, E4M3, F16, F32, CommOptions as _CommOptions, FabricError, MeshError,
                   Shape4, ShapeError, InvalidArgument, FuspError, check, lib)

_DT = {torch.float32: F32, torch.float16: F16, torch.bfloat16: BF16}
_TORCH = {F32: torch.float32, F16: torch.float16, BF16: torch.bfloat16}

kFp8Max = 448.0       # fp8.hpp:15
kFp8MaxCode = 0x7E    # fp8.hpp:16
kFp8NanCode = 0x7F    # fp8.hpp:17


def _ptr(t: Optional[torch.Tensor]):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _dev(t: torch.Tensor) -> torch.Tensor:
    if not t.is_cuda:
        raise InvalidArgument(4, "fastusp operates on CUDA tensors (no CPU fallback)")
    return t.contiguous()


def _shape4(t: torch.Tensor) -> Shape4:
    if t.dim() != 4:
        raise ShapeError(1, f"expected a rank-4 [B,H,S,D] tensor, got {tuple(t.shape)}")
    return Shape4(*[int(x) for x in t.shape])


# ---- fp8 (fp8.hpp:23-49) ----------------------------------------------------------------
def encode_e4m3(x: torch.Tensor) -> torch.Tensor:
    """encode_e4m3 (fp8.cpp:45-68) elementwise on a float32 CUDA tensor."""
    x = _dev(x).float()
    out = torch.empty(x.shape, dtype=torch.uint8, device=x.device)
    check(lib().fusp_encode_e4m3(_ptr(x), x.numel(), _ptr(out), _stream()))
    return out


def decode_e4m3(codes: torch.Tensor) -> torch.Tensor:
    """decode_e4m3 (fp8.cpp:39-43) elementwise."""
    codes = _dev(codes)
    out = torch.empty(codes.shape, dtype=torch.float32, device=codes.device)
    check(lib().fusp_decode_e4m3(_ptr(codes), codes.numel(), _ptr(out), _stream()))
    return out


@dataclass
class QuantizedTensor:
    """= uspsim::QuantizedTensor (fp8.hpp:30-42): codes + one device-resident f32 scale."""
    codes: torch.Tensor
    scale_dev: torch.Tensor

    @property
    def scale(self) -> float:
        return float(self.scale_dev.item())

    def shape(self):
        return tuple(self.codes.shape)

    def slice_heads(self, h0: int, count: int) -> "QuantizedTensor":
        """fp8.cpp:100-105: head slice keeps the tensor-wide scale."""
        return QuantizedTensor(self.codes[:, h0:h0 + count].contiguous(), self.scale_dev)


def quantize(x: torch.Tensor, check_finite: bool = True) -> QuantizedTensor:
    """quantize (fp8.cpp:107-123): bit-exact codes and scale; raises InvalidArgument on non-finite."""
    x = _dev(x)
    if x.dtype not in _DT:
        x = x.float()
    codes = torch.empty(x.shape, dtype=torch.uint8, device=x.device)
    scale = torch.empty(1, dtype=torch.float32, device=x.device)
    check(lib().fusp_quantize_e4m3(_ptr(x), _DT[x.dtype], x.numel(), _ptr(codes), _ptr(scale),
                                   int(check_finite), _stream()))
    return QuantizedTensor(codes, scale)


def dequantize(q: QuantizedTensor, dtype=torch.float32) -> torch.Tensor:
    """dequantize (fp8.cpp:125-130): decode(code) * scale."""
    out = torch.empty(q.codes.shape, dtype=dtype, device=q.codes.device)
    check(lib().fusp_dequantize_e4m3(_ptr(q.codes), _ptr(q.scale_dev), q.codes.numel(), _ptr(out),
                                     _DT[dtype], _stream()))
    return out


# ---- attention numerics (tensor.hpp:64-98) -----------------------------------------------
@dataclass
class AttnResult:
    """= uspsim::AttnResultT (tensor.hpp:75-83): out [B,H,Sq,D], lse [B,H,Sq] (natural log)."""
    out: torch.Tensor
    lse: torch.Tensor

    @staticmethod
    def identity(shape, device="cuda") -> "AttnResult":
        """tensor.cpp:110-117: O = 0, lse = -inf."""
        b, h, s, d = shape
        return AttnResult(torch.zeros(shape, device=device),
                          torch.full((b, h, s), float("-inf"), device=device))


def _check_qkv(q, k, v):
    """check_qkv (tensor.cpp:121-139): same messages, ShapeError."""
    if not (q.shape[0] == k.shape[0] == v.shape[0]):
        raise ShapeError(1, f"attention: batch axis mismatch, Q B={q.shape[0]} K B={k.shape[0]} "
                            f"V B={v.shape[0]}")
    if not (q.shape[1] == k.shape[1] == v.shape[1]):
        raise ShapeError(1, f"attention: head axis mismatch, Q H={q.shape[1]} K H={k.shape[1]} "
                            f"V H={v.shape[1]}")
    if not (q.shape[3] == k.shape[3] == v.shape[3]):
        raise ShapeError(1, f"attention: head-dim axis mismatch, Q D={q.shape[3]} K D={k.shape[3]} "
                            f"V D={v.shape[3]}")
    if k.shape[2] != v.shape[2]:
        raise ShapeError(1, f"attention: sequence axis mismatch between K S={k.shape[2]} and "
                            f"V S={v.shape[2]}")


def attention_with_lse(q, k, v, out_dtype=torch.float32) -> AttnResult:
    """attention_with_lse (tensor.cpp:193-202) on the tcgen05 kernel."""
    q, k, v = _dev(q), _dev(k), _dev(v)
    for t in (q, k, v):
        _shape4(t)
    _check_qkv(q, k, v)
    dt = q.dtype if q.dtype in _DT else torch.float32
    q, k, v = q.to(dt), k.to(dt), v.to(dt)
    b, h, sq, d = q.shape
    out = torch.empty((b, h, sq, d), dtype=out_dtype, device=q.device)
    lse = torch.empty((b, h, sq), dtype=torch.float32, device=q.device)
    check(lib().fusp_attention_with_lse(_ptr(q), _ptr(k), _ptr(v), _DT[dt], _shape4(q),
                                        int(k.shape[2]), _ptr(out), _DT[out_dtype], _ptr(lse),
                                        _stream()))
    return AttnResult(out, lse)


def attention_reference(q, k, v, out_dtype=torch.float32) -> torch.Tensor:
    """attention_reference (tensor.cpp:185-191): attention_with_lse without the LSE."""
    return attention_with_lse(q, k, v, out_dtype).out


def merge_lse(a: AttnResult, b: AttnResult) -> AttnResult:
    """merge_lse (tensor.cpp:204-243)."""
    if tuple(a.out.shape) != tuple(b.out.shape):
        raise ShapeError(1, f"merge_lse: output shapes differ, {list(a.out.shape)} vs "
                            f"{list(b.out.shape)}")
    if a.lse.numel() != b.lse.numel():
        raise ShapeError(1, f"merge_lse: lse lengths differ, {a.lse.numel()} vs {b.lse.numel()}")
    o1, o2 = _dev(a.out).float(), _dev(b.out).float()
    l1, l2 = _dev(a.lse).float(), _dev(b.lse).float()
    out = torch.empty_like(o1)
    lse = torch.empty_like(l1)
    check(lib().fusp_merge_lse(_ptr(o1), _ptr(l1), _ptr(o2), _ptr(l2), _shape4(o1), _ptr(out),
                               _ptr(lse), _stream()))
    return AttnResult(out, lse)


# ---- mesh (mesh.hpp:27-50) -----------------------------------------------------------------
@dataclass
class ProcessGroup:
    """= uspsim::ProcessGroup (fabric.hpp:20-28)."""
    members: List[int]

    def size(self) -> int:
        return len(self.members)

    def position_of(self, rank: int) -> int:
        return self.members.index(rank) if rank in self.members else -1

    def key(self) -> str:
        return ",".join(str(m) for m in self.members)


@dataclass
class Mesh2D:
    """= uspsim::Mesh2D (mesh.hpp:27-41): rank = ring_index * U + ulysses_index."""
    n: int = 1
    r: int = 1
    u: int = 1
    ring_groups: List[ProcessGroup] = field(default_factory=list)
    ulysses_groups: List[ProcessGroup] = field(default_factory=list)

    def ring_index(self, rank: int) -> int:
        return rank // self.u

    def ulysses_index(self, rank: int) -> int:
        return rank % self.u

    def ring_group(self, rank: int) -> ProcessGroup:
        if rank < 0 or rank >= self.n:
            raise MeshError(2, f"rank {rank} out of range")
        return self.ring_groups[self.ulysses_index(rank)]

    def ulysses_group(self, rank: int) -> ProcessGroup:
        if rank < 0 or rank >= self.n:
            raise MeshError(2, f"rank {rank} out of range")
        return self.ulysses_groups[self.ring_index(rank)]

    def to_json(self) -> dict:
        return {"workers": self.n, "ring_dim": self.r, "ulysses_dim": self.u,
                "ring_groups": [g.members for g in self.ring_groups],
                "ulysses_groups": [g.members for g in self.ulysses_groups]}


def make_mesh(n: int, r: int) -> Mesh2D:
    """make_mesh (mesh.cpp:34-55)."""
    ug = (ctypes.c_int * max(n, 1))()
    rg = (ctypes.c_int * max(n, 1))()
    check(lib().fusp_mesh_make(n, r, ug, rg))
    u = n // r
    return Mesh2D(n, r, u,
                  ring_groups=[ProcessGroup(list(rg[j * r:(j + 1) * r])) for j in range(u)],
                  ulysses_groups=[ProcessGroup(list(ug[i * u:(i + 1) * u])) for i in range(r)])


def build_mesh(n: int, max_ring_dim_size: int, heads: int) -> Mesh2D:
    """build_mesh (mesh.cpp:57-79): the largest feasible R <= max_ring_dim_size."""
    r, u = ctypes.c_int(), ctypes.c_int()
    check(lib().fusp_mesh_build(n, max_ring_dim_size, heads, ctypes.byref(r), ctypes.byref(u)))
    return make_mesh(n, r.value)


def kernel_launch_count() -> int:
    return int(lib().fusp_kernel_launch_count())

"""Python host mirror of the reference uspsim API, over the fastusp C ABI.

Names, argument meanings and error classes follow the reference
(/root/reference/proj/include/uspsim/{tensor,fp8,mesh,protocols}.hpp); tensors
are torch CUDA tensors (device memory plumbing only -- every computation runs in
libfastusp.so's sm_100a kernels).
"""
from __future__ import annotations

import contextlib
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


def quantize_blocks(x: torch.Tensor, block: int):
    """Per-block quantize (B200 extension): each run of `block` elements is quantized like
    uspsim::quantize on that slice alone.  Returns (codes, scales[numel // block])."""
    x = _dev(x)
    if x.dtype not in _DT:
        x = x.float()
    codes = torch.empty(x.shape, dtype=torch.uint8, device=x.device)
    scales = torch.empty(max(x.numel() // max(block, 1), 1), dtype=torch.float32, device=x.device)
    check(lib().fusp_quantize_e4m3_blocks(_ptr(x), _DT[x.dtype], x.numel(), block, _ptr(codes),
                                          _ptr(scales), _stream()))
    return codes, scales


def dequantize_blocks(codes: torch.Tensor, scales: torch.Tensor, block: int,
                      dtype=torch.float32) -> torch.Tensor:
    out = torch.empty(codes.shape, dtype=dtype, device=codes.device)
    check(lib().fusp_dequantize_e4m3_blocks(_ptr(codes), _ptr(scales), codes.numel(), block,
                                            _ptr(out), _DT[dtype], _stream()))
    return out


def requantize(codes: torch.Tensor, seg_scales: torch.Tensor, seg: int) -> QuantizedTensor:
    """Ring-hop re-quantization (protocols.cpp:113-115, 309-310): quantize(dequantize(chunk))
    where every run of `seg` codes carries its own scale seg_scales[i // seg].  Bit-exact."""
    codes, seg_scales = _dev(codes), _dev(seg_scales).float().contiguous()
    out = torch.empty(codes.shape, dtype=torch.uint8, device=codes.device)
    scale = torch.empty(1, dtype=torch.float32, device=codes.device)
    check(lib().fusp_requantize_e4m3(_ptr(codes), _ptr(seg_scales), codes.numel(), seg, _ptr(out),
                                     _ptr(scale), _stream()))
    return QuantizedTensor(out, scale)


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
    q, k = q.to(dt), k.to(dt)
    vdt = v.dtype if v.dtype in _DT else torch.float32
    v = v.to(vdt)
    b, h, sq, d = q.shape
    out = torch.empty((b, h, sq, d), dtype=out_dtype, device=q.device)
    lse = torch.empty((b, h, sq), dtype=torch.float32, device=q.device)
    check(lib().fusp_attention_with_lse_ex(_ptr(q), _ptr(k), _ptr(v), _DT[dt], _DT[vdt],
                                           _shape4(q), int(k.shape[2]), _ptr(out), _DT[out_dtype],
                                           _ptr(lse), _stream()))
    return AttnResult(out, lse)


def stage_f16(x: torch.Tensor):
    """Range-guarded f16 staging (fusp_stage_f16): x [..., rows, 128] viewed as [heads][rows][128]
    -> (y f16, exps int32 [heads]) with x = y * 2^exps exactly (fastusp_internal.h)."""
    x = _dev(x)
    if x.dtype not in _DT:
        x = x.float()
    heads = x.numel() // (x.shape[-2] * x.shape[-1])
    y = torch.empty(x.shape, dtype=torch.float16, device=x.device)
    exps = torch.empty(heads, dtype=torch.int32, device=x.device)
    check(lib().fusp_stage_f16(_ptr(x), _DT[x.dtype], heads, x.shape[-2], _ptr(y), _ptr(exps),
                               _stream()))
    return y, exps


_SCHEDULES = {"auto": 0, "whole": 1, "split": 2, "aligned": 3, "kv2": 4, "kv2split": 5}


@contextlib.contextmanager
def attention_schedule(mode: str = "auto", max_ctas: int = 0):
    """Pin the attention kernel's work schedule inside the block (tests, benchmarks):
    "whole" = one 256-row q-block per CTA turn, "split" = stream-K over (q-block, KV tile)
    units, "auto" = split only when whole q-blocks leave SMs idle; `max_ctas` caps the
    persistent grid (0 = every SM)."""
    check(lib().fusp_attention_schedule(_SCHEDULES[mode], int(max_ctas)))
    try:
        yield
    finally:
        check(lib().fusp_attention_schedule(0, 0))


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


# ---- communication options (protocols.hpp:12-15) ----------------------------------------------
@dataclass
class CommOptions:
    """= uspsim::CommOptions plus B200 extensions (out_dtype, check_finite, fp8_block)."""
    fp8_kv: bool = False
    pipelined_ring: bool = False
    out_dtype: torch.dtype = torch.float32
    check_finite: bool = True
    fp8_block: int = 0

    def _c(self) -> _CommOptions:
        return _CommOptions(int(self.fp8_kv), int(self.pipelined_ring), _DT[self.out_dtype],
                            int(self.check_finite), int(self.fp8_block))


# ---- per-rank contexts (fabric.hpp:136-166) ------------------------------------------------------
class Fabric:
    """In-process fabric: `world` ranks living in this process (threads as ranks)."""

    def __init__(self, world: int):
        h = ctypes.c_void_p()
        check(lib().fusp_fabric_create(world, ctypes.byref(h)))
        self.handle = h
        self.world = world

    def close(self):
        if self.handle:
            lib().fusp_fabric_destroy(self.handle)
            self.handle = None


class WorkerContext:
    """= uspsim::WorkerContext: one rank, bound to one CUDA device."""

    def __init__(self, handle, device: int):
        self.handle = handle
        self.device = device

    @classmethod
    def local(cls, fabric: Fabric, rank: int, device: int = 0) -> "WorkerContext":
        h = ctypes.c_void_p()
        check(lib().fusp_ctx_create_local(fabric.handle, rank, device, ctypes.byref(h)))
        return cls(h, device)

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (ctypes.c_uint8 * 128)()
        check(lib().fusp_nccl_unique_id(buf))
        return bytes(buf)

    @classmethod
    def nccl(cls, uid: bytes, world: int, rank: int, device: int) -> "WorkerContext":
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        h = ctypes.c_void_p()
        check(lib().fusp_ctx_create_nccl(buf, world, rank, device, ctypes.byref(h)))
        return cls(h, device)

    def rank(self) -> int:
        return lib().fusp_ctx_rank(self.handle)

    def create_group(self, members) -> ctypes.c_void_p:
        """fusp_group_create: a ProcessGroup handle on this context, cached by member list.
        Collective over the world for NCCL contexts (every rank calls, members=[] to opt out)."""
        key = tuple(int(m) for m in members)
        cache = self.__dict__.setdefault("_groups", {})
        if key in cache:
            return cache[key]
        arr = (ctypes.c_int * max(len(key), 1))(*key)
        h = ctypes.c_void_p()
        check(lib().fusp_group_create(self.handle, arr, len(key), ctypes.byref(h)))
        if key:
            cache[key] = h
        return h

    def world_size(self) -> int:
        return lib().fusp_ctx_world(self.handle)

    def traffic(self):
        """(all_to_all bytes, send bytes) this rank put on the wire (TrafficLog::bytes_for)."""
        a, s = ctypes.c_uint64(), ctypes.c_uint64()
        check(lib().fusp_ctx_traffic(self.handle, ctypes.byref(a), ctypes.byref(s)))
        return a.value, s.value

    def reset_traffic(self):
        check(lib().fusp_ctx_reset_traffic(self.handle))

    def _json(self, fn):
        import json
        n = ctypes.c_size_t()
        check(fn(self.handle, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value + 1)
        check(fn(self.handle, buf, n.value + 1, ctypes.byref(n)))
        return json.loads(buf.value.decode())

    def traffic_log(self) -> list:
        """TrafficLog::to_json entries of this rank (fabric.cpp:72-87)."""
        return self._json(lib().fusp_ctx_traffic_json)

    def timeline(self) -> list:
        """Timeline::to_json of the last layer call, with device timestamps t_ms."""
        return self._json(lib().fusp_ctx_timeline_json)

    def debug_wire(self, enable: bool = True):
        """fusp_ctx_debug_wire: record every payload this rank puts on the wire (eager calls)."""
        check(lib().fusp_ctx_debug_wire(self.handle, int(enable)))

    def wire_records(self):
        """[(kind, round, bytes as np.uint8)]: kind 0 Ulysses-in send slots, 1/2 ring K/V part."""
        import numpy as np
        out = []
        for i in range(lib().fusp_ctx_debug_wire_count(self.handle)):
            kind, rnd, n = ctypes.c_int(), ctypes.c_int(), ctypes.c_size_t()
            check(lib().fusp_ctx_debug_wire_get(self.handle, i, ctypes.byref(kind), ctypes.byref(rnd),
                                                None, 0, ctypes.byref(n)))
            buf = np.empty(n.value, np.uint8)
            check(lib().fusp_ctx_debug_wire_get(self.handle, i, None, None,
                                                buf.ctypes.data_as(ctypes.c_void_p), n.value, None))
            out.append((kind.value, rnd.value, buf))
        return out

    def enable_peer_memory(self, window_bytes: int):
        """fusp_ctx_peer_enable (collective over the world): the Ulysses reshards of later
        layers are fused into the pack kernel and the attention epilogue, which store straight
        into the members' windows (NVLink / NVSwitch peer memory); see fastusp.h."""
        check(lib().fusp_ctx_peer_enable(self.handle, int(window_bytes)))

    def peer_window(self, window_bytes: int) -> bytes:
        """Two-step form (own bootstrap): create this rank's window, return its handle."""
        buf = (ctypes.c_uint8 * 128)()
        check(lib().fusp_ctx_peer_window(self.handle, int(window_bytes), buf))
        return bytes(buf)

    def peer_open(self, handles) -> None:
        """Map the world's window handles (rank order) created by peer_window."""
        blob = b"".join(handles)
        buf = (ctypes.c_uint8 * len(blob)).from_buffer_copy(blob)
        check(lib().fusp_ctx_peer_open(self.handle, buf))

    def disable_peer_memory(self) -> None:
        """fusp_ctx_peer_disable: back to the backend transport (every rank of a group)."""
        check(lib().fusp_ctx_peer_disable(self.handle))

    def peer_stats(self):
        """(layers on the peer path, layers that fell back to the backend) since enabling."""
        a, b = ctypes.c_uint64(), ctypes.c_uint64()
        check(lib().fusp_ctx_peer_stats(self.handle, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def synchronize(self, stream=None, timeout_s: float = 0.0):
        """fusp_ctx_synchronize: bounded host wait; a stalled / failed peer raises
        DeadlockError (the NCCL communicators are aborted) instead of hanging."""
        check(lib().fusp_ctx_synchronize(self.handle, _stream(stream), float(timeout_s)))

    def ring_timings(self, max_steps: int = 32):
        """Per ring step device times (ms) of the last call: (compute[], comm[])."""
        c = (ctypes.c_float * max_steps)()
        m = (ctypes.c_float * max_steps)()
        n = ctypes.c_int()
        check(lib().fusp_ctx_ring_timings(self.handle, max_steps, c, m, ctypes.byref(n)))
        return list(c[:n.value]), list(m[:n.value])

    def close(self):
        if self.handle:
            for h in self.__dict__.pop("_groups", {}).values():
                lib().fusp_group_destroy(h)
            lib().fusp_ctx_destroy(self.handle)
            self.handle = None


def peer_window_bytes(world: int, ring_dim: int, local_shape, dtype=torch.bfloat16,
                      opts: Optional["CommOptions"] = None) -> int:
    """fusp_peer_window_bytes: window bytes a USP layer of this local shape [B,H,S/N,D] needs
    on every member."""
    o = opts or CommOptions()
    n = ctypes.c_size_t()
    check(lib().fusp_peer_window_bytes(world, ring_dim, _DT[dtype], Shape4(*local_shape),
                                       ctypes.byref(o._c()), ctypes.byref(n)))
    return n.value


@dataclass
class RunReport:
    results: list
    traffic: list  # per rank (all_to_all bytes, send bytes)


def run_protocol(n_workers: int, program: Callable[[WorkerContext], object], device: int = 0,
                 devices: Optional[List[int]] = None) -> RunReport:
    """= uspsim::run_protocol (fabric.hpp:180): one host thread per rank, each with its own
    CUDA stream; ranks may share a device.  Raises the first rank's exception."""
    if n_workers < 1:
        raise FabricError(3, "run_protocol: need at least one worker")
    fab = Fabric(n_workers)
    devs = devices or [device] * n_workers
    ctxs = [WorkerContext.local(fab, r, devs[r]) for r in range(n_workers)]
    results = [None] * n_workers
    errors = [None] * n_workers

    def body(r):
        try:
            torch.cuda.set_device(devs[r])
            s = torch.cuda.Stream(device=devs[r])
            with torch.cuda.stream(s):
                results[r] = program(ctxs[r])
            s.synchronize()
        except BaseException as e:  # noqa: BLE001 -- re-raised below
            errors[r] = e

    try:
        if n_workers == 1:
            body(0)
        else:
            th = [threading.Thread(target=body, args=(r,)) for r in range(n_workers)]
            for t in th:
                t.start()
            for t in th:
                t.join()
        for e in errors:
            if e is not None:
                raise e
        return RunReport(results, [c.traffic() for c in ctxs])
    finally:
        for c in ctxs:
            c.close()
        fab.close()


# ---- protocols (protocols.hpp:28-71) --------------------------------------------------------------
def split_sequence(full: torch.Tensor, count: int) -> List[torch.Tensor]:
    """split_sequence (protocols.cpp:10-21)."""
    if count < 1:
        raise ShapeError(1, "split_sequence: count must be >= 1")
    s = full.shape[2]
    if s % count:
        raise ShapeError(1, f"split_sequence: S={s} not divisible by shard count {count}")
    c = s // count
    return [full[:, :, i * c:(i + 1) * c].contiguous() for i in range(count)]


def gather_output(shards: List[torch.Tensor]) -> torch.Tensor:
    """gather_output (protocols.cpp:23): concatenation along S in rank order."""
    return torch.cat(list(shards), dim=2)


def _check_local(q, k, v, where):
    if not (tuple(q.shape) == tuple(k.shape) == tuple(v.shape)):
        raise ShapeError(1, f"{where}: local Q/K/V shapes differ: Q={list(q.shape)} "
                            f"K={list(k.shape)} V={list(v.shape)}")
    if q.dtype != k.dtype or q.dtype != v.dtype:
        raise InvalidArgument(4, f"{where}: Q/K/V dtypes differ")


def _inputs(q, k, v, where):
    q, k, v = _dev(q), _dev(k), _dev(v)
    _shape4(q)
    _check_local(q, k, v, where)
    if q.dtype not in _DT:
        q, k, v = q.float(), k.float(), v.float()
    return q, k, v


@dataclass
class QKPrologue:
    """MMDiT QK RMSNorm + RoPE fused into the Ulysses pack (fusp_qk_prologue in fastusp.h).
    Weights [D] and tables [rows][D/2] are f32 CUDA tensors; None skips that step.
    rope_pos0 = -1: this rank's first row sits at position rank * S_local."""
    q_norm_weight: Optional[torch.Tensor] = None
    k_norm_weight: Optional[torch.Tensor] = None
    eps: float = 1e-6
    rope_cos: Optional[torch.Tensor] = None
    rope_sin: Optional[torch.Tensor] = None
    rope_pos0: int = -1

    def _c(self) -> "_lib.QKPrologue":
        def f32(t):
            if t is None:
                return None
            if t.dtype != torch.float32 or not t.is_cuda or not t.is_contiguous():
                raise InvalidArgument(4, "QKPrologue tensors must be contiguous f32 CUDA tensors")
            return t
        qw, kw, c, s = (f32(t) for t in (self.q_norm_weight, self.k_norm_weight,
                                         self.rope_cos, self.rope_sin))
        rows = c.shape[0] if c is not None else 0
        return _lib.QKPrologue(_ptr(qw), _ptr(kw), float(self.eps), _ptr(c), _ptr(s), rows,
                               int(self.rope_pos0))


def rope_tables(positions: int, d: int = 128, theta: float = 10000.0, device="cuda"):
    """cos/sin [positions][d/2] f32 for frequencies theta^(-2i/d) (1-axis RoPE)."""
    inv = theta ** (-torch.arange(0, d, 2, dtype=torch.float64) / d)
    ang = torch.arange(positions, dtype=torch.float64)[:, None] * inv[None, :]
    return (ang.cos().float().to(device).contiguous(), ang.sin().float().to(device).contiguous())


def usp_attention(ctx: WorkerContext, q, k, v, mesh: Mesh2D,
                  opts: Optional[CommOptions] = None,
                  prologue: Optional[QKPrologue] = None) -> torch.Tensor:
    """usp_attention (protocols.cpp:321-340): local shards [B,H,S/N,D] -> [B,H,S/N,D].
    `prologue` (B200 extension): QK RMSNorm + RoPE applied inside the Ulysses pack."""
    opts = opts or CommOptions()
    if mesh.n != ctx.world_size():
        raise MeshError(2, f"mesh covers {mesh.n} workers but the fabric has {ctx.world_size()}")
    q, k, v = _inputs(q, k, v, "usp")
    out = torch.empty(q.shape, dtype=opts.out_dtype, device=q.device)
    co = opts._c()
    if prologue is None:
        check(lib().fusp_usp_attention(ctx.handle, mesh.r, _ptr(q), _ptr(k), _ptr(v),
                                       _DT[q.dtype], _shape4(q), _ptr(out), ctypes.byref(co),
                                       _stream()))
    else:
        pc = prologue._c()
        check(lib().fusp_usp_attention_ex(ctx.handle, mesh.r, _ptr(q), _ptr(k), _ptr(v),
                                          _DT[q.dtype], _shape4(q), _ptr(out), ctypes.byref(co),
                                          ctypes.byref(pc), _stream()))
    return out


def usp_attention_with_lse(ctx: WorkerContext, q, k, v, mesh: Mesh2D,
                           opts: Optional[CommOptions] = None) -> AttnResult:
    """usp_attention that also returns the rows' natural-log LSE [B,H,S/N] (fusp_usp_attention_lse;
    the reference drops it, protocols.cpp:339)."""
    opts = opts or CommOptions()
    if mesh.n != ctx.world_size():
        raise MeshError(2, f"mesh covers {mesh.n} workers but the fabric has {ctx.world_size()}")
    q, k, v = _inputs(q, k, v, "usp")
    out = torch.empty(q.shape, dtype=opts.out_dtype, device=q.device)
    lse = torch.empty(q.shape[:3], dtype=torch.float32, device=q.device)
    co = opts._c()
    check(lib().fusp_usp_attention_lse(ctx.handle, mesh.r, _ptr(q), _ptr(k), _ptr(v), _DT[q.dtype],
                                       _shape4(q), _ptr(out), _ptr(lse), ctypes.byref(co),
                                       _stream()))
    return AttnResult(out, lse)


def _group_handle(ctx: WorkerContext, group: Optional[ProcessGroup]):
    """The fusp_group of `group` on this context (NULL for the world in rank order).  Created on
    first use -- for NCCL contexts group creation is collective over the world, so create
    those groups up front on every rank with ctx.create_group(members)."""
    if group is None or list(group.members) == list(range(ctx.world_size())):
        return ctypes.c_void_p(0)
    return ctx.create_group(group.members)


def ulysses_attention(ctx: WorkerContext, q, k, v, group: Optional[ProcessGroup] = None,
                      opts: Optional[CommOptions] = None, return_lse: bool = False):
    """ulysses_attention(ctx, q, k, v, group, opts) (protocols.cpp:207-214); group None = world.
    return_lse: an AttnResult with the rows' LSE (B200 extension)."""
    opts = opts or CommOptions()
    q, k, v = _inputs(q, k, v, "ulysses")
    out = torch.empty(q.shape, dtype=opts.out_dtype, device=q.device)
    lse = torch.empty(q.shape[:3], dtype=torch.float32, device=q.device) if return_lse else None
    co = opts._c()
    check(lib().fusp_ulysses_attention_group(ctx.handle, _group_handle(ctx, group), _ptr(q), _ptr(k),
                                             _ptr(v), _DT[q.dtype], _shape4(q), _ptr(out), _ptr(lse),
                                             ctypes.byref(co), _stream()))
    return AttnResult(out, lse) if return_lse else out


def _ring(ctx, q, k, v, group, opts, pipelined):
    opts = opts or CommOptions()
    q, k, v = _inputs(q, k, v, "ring")
    out = torch.empty(q.shape, dtype=opts.out_dtype, device=q.device)
    lse = torch.empty(q.shape[:3], dtype=torch.float32, device=q.device)
    co = opts._c()
    co.pipelined_ring = int(pipelined)
    check(lib().fusp_ring_attention_group(ctx.handle, _group_handle(ctx, group), _ptr(q), _ptr(k),
                                          _ptr(v), _DT[q.dtype], _shape4(q), _ptr(out), _ptr(lse),
                                          ctypes.byref(co), _stream()))
    return AttnResult(out, lse)


def ring_attention_serial(ctx, q, k, v, group=None, opts=None) -> AttnResult:
    """ring_attention_serial (protocols.cpp:237-268) over `group` (None = world)."""
    return _ring(ctx, q, k, v, group, opts, False)


def ring_attention_pipelined(ctx, q, k, v, group=None, opts=None) -> AttnResult:
    """ring_attention_pipelined (protocols.cpp:270-319): double-buffered on a side stream."""
    return _ring(ctx, q, k, v, group, opts, True)


@dataclass
class Resharded:
    """= uspsim::detail::Resharded (protocols.hpp:77-79): [B, H/U, U*S_local, D]."""
    q: torch.Tensor
    k: torch.Tensor
    v: torch.Tensor


class detail:  # noqa: N801 -- namespace mirroring uspsim::detail (protocols.hpp:73-95)
    @staticmethod
    def ulysses_input_reshard(ctx: WorkerContext, q, k, v, group: Optional[ProcessGroup] = None,
                              opts: Optional[CommOptions] = None,
                              out_dtype=torch.float32) -> Resharded:
        """detail::ulysses_input_reshard (protocols.cpp:125-180) on the GPU path: pack ->
        all_to_all -> unpack; FP8 K/V come back as the exact dequantized values."""
        opts = opts or CommOptions()
        q, k, v = _inputs(q, k, v, "ulysses")
        gh = _group_handle(ctx, group)
        u = len(group.members) if group is not None else ctx.world_size()
        b, h, s, d = q.shape
        if h % u:
            raise ShapeError(1, f"ulysses: head count H={h} not divisible by ulysses dimension U={u}")
        shp = (b, h // u, s * u, d)
        outs = [torch.empty(shp, dtype=out_dtype, device=q.device) for _ in range(3)]
        co = opts._c()
        check(lib().fusp_ulysses_input_reshard(ctx.handle, gh, _ptr(q), _ptr(k), _ptr(v),
                                               _DT[q.dtype], _shape4(q), _ptr(outs[0]),
                                               _ptr(outs[1]), _ptr(outs[2]), _DT[out_dtype],
                                               ctypes.byref(co), _stream()))
        return Resharded(*outs)

    @staticmethod
    def ulysses_output_reshard(ctx: WorkerContext, out, group: Optional[ProcessGroup] = None):
        """detail::ulysses_output_reshard (protocols.cpp:182-203): [B,H/U,S,D] -> [B,H,S/U,D]."""
        o = _dev(out)
        if o.dtype not in _DT:
            o = o.float()
        u = len(group.members) if group is not None else ctx.world_size()
        b, hp, s, d = o.shape
        if s % u:
            raise ShapeError(1, f"ulysses: gathered sequence length S={s} not divisible by ulysses "
                                f"dimension U={u}")
        res = torch.empty((b, hp * u, s // u, d), dtype=o.dtype, device=o.device)
        check(lib().fusp_ulysses_output_reshard(ctx.handle, _group_handle(ctx, group), _ptr(o),
                                                _DT[o.dtype], _shape4(o), _ptr(res), _stream()))
        return res


def out_projection(o: torch.Tensor, w: torch.Tensor, out_dtype=torch.bfloat16) -> torch.Tensor:
    """The joint-attention block's output projection on the tcgen05 GEMM (fusp_out_projection):
    o [B,H,S,128] (bf16|f16, the layer's output layout) x w [H*128, N] -> y [B,S,N]."""
    o, w = _dev(o), _dev(w)
    b, h, s_, d = _shape4(o).b, o.shape[1], o.shape[2], o.shape[3]
    if w.dim() != 2 or w.shape[0] != h * d:
        raise ShapeError(1, f"out_projection: w must be [{h * d}, N], got {list(w.shape)}")
    y = torch.empty(b, s_, w.shape[1], dtype=out_dtype, device=o.device)
    check(lib().fusp_out_projection(_ptr(o), _DT[o.dtype], _shape4(o), _ptr(w), int(w.shape[1]),
                                    _ptr(y), _DT[out_dtype], _stream()))
    return y


def usp_attention_proj(ctx: WorkerContext, q, k, v, mesh: Mesh2D, w_out: torch.Tensor,
                       opts: Optional[CommOptions] = None, prologue: Optional[QKPrologue] = None,
                       out_dtype=torch.bfloat16):
    """usp_attention then the output projection in one C-ABI call (fusp_usp_attention_proj).
    opts.out_dtype (bf16|f16) is the attention output that feeds the projection."""
    opts = opts or CommOptions(out_dtype=torch.bfloat16)
    if mesh.n != ctx.world_size():
        raise MeshError(2, f"mesh covers {mesh.n} workers but the fabric has {ctx.world_size()}")
    q, k, v = _inputs(q, k, v, "usp")
    w_out = _dev(w_out)
    attn = torch.empty(q.shape, dtype=opts.out_dtype, device=q.device)
    y = torch.empty(q.shape[0], q.shape[2], w_out.shape[1], dtype=out_dtype, device=q.device)
    co = opts._c()
    pc = prologue._c() if prologue is not None else None
    check(lib().fusp_usp_attention_proj(ctx.handle, mesh.r, _ptr(q), _ptr(k), _ptr(v), _DT[q.dtype],
                                        _shape4(q), _ptr(attn), ctypes.byref(co),
                                        ctypes.byref(pc) if pc is not None else None,
                                        _ptr(w_out), int(w_out.shape[1]), _ptr(y), _DT[out_dtype],
                                        _stream()))
    return y


def usp_block(ctx: WorkerContext, x: torch.Tensor, w_qkv: torch.Tensor, heads: int,
              w_out: torch.Tensor, mesh: Mesh2D, prologue: Optional[QKPrologue] = None,
              opts: Optional[CommOptions] = None, out_dtype=torch.bfloat16) -> torch.Tensor:
    """The MMDiT joint-attention block on this rank's tokens (fusp_usp_block): x [B,S/N,C]
    -> QKV projection (+ QK RMSNorm / RoPE in its epilogue) -> USP layer -> output projection
    -> y [B,S/N,N]."""
    opts = opts or CommOptions(check_finite=False)
    if mesh.n != ctx.world_size():
        raise MeshError(2, f"mesh covers {mesh.n} workers but the fabric has {ctx.world_size()}")
    x, w_qkv, w_out = _dev(x), _dev(w_qkv), _dev(w_out)
    if x.dim() != 3:
        raise ShapeError(1, f"usp_block: x must be [B, S, C], got {list(x.shape)}")
    b, s_, c = x.shape
    if tuple(w_qkv.shape) != (c, 3 * heads * 128) or w_out.dim() != 2 or w_out.shape[0] != heads * 128:
        raise ShapeError(1, f"usp_block: w_qkv must be [{c}, {3 * heads * 128}] and w_out "
                            f"[{heads * 128}, N]; got {list(w_qkv.shape)}, {list(w_out.shape)}")
    y = torch.empty(b, s_, w_out.shape[1], dtype=out_dtype, device=x.device)
    co = opts._c()
    pc = prologue._c() if prologue is not None else None
    check(lib().fusp_usp_block(ctx.handle, mesh.r, _ptr(x), _DT[x.dtype], b, s_, c, _ptr(w_qkv),
                               heads, ctypes.byref(pc) if pc is not None else None, _ptr(w_out),
                               int(w_out.shape[1]), _ptr(y), _DT[out_dtype], ctypes.byref(co),
                               _stream()))
    return y


def usp_attention_host(ctx: WorkerContext, q, k, v, mesh: Mesh2D,
                       opts: Optional[CommOptions] = None, out=None):
    """usp_attention on HOST tensors (H2D, layer, D2H inside one C-ABI call, pipelined over
    head chunks).  Pinned q/k/v/out overlap the copies with the compute; `out` may be a
    preallocated host tensor of the output dtype (default: a new pinned one)."""
    opts = opts or CommOptions()
    if q.is_cuda:
        raise InvalidArgument(4, "usp_attention_host expects host tensors")
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    _check_local(q, k, v, "usp")
    if out is None:
        out = torch.empty(q.shape, dtype=opts.out_dtype, pin_memory=torch.cuda.is_available())
    elif out.is_cuda or tuple(out.shape) != tuple(q.shape) or out.dtype != opts.out_dtype \
            or not out.is_contiguous():
        raise InvalidArgument(4, "usp_attention_host: out must be a contiguous host tensor "
                                 f"{list(q.shape)} of {opts.out_dtype}")
    co = opts._c()
    check(lib().fusp_usp_attention_host(ctx.handle, mesh.r, _ptr(q), _ptr(k), _ptr(v),
                                        _DT[q.dtype], _shape4(q), _ptr(out), ctypes.byref(co),
                                        _stream()))
    return out


class BlockGraph:
    """CUDA graph of `layers` back-to-back usp_block calls (fusp_graph_capture_block): the QKV
    projection, the USP layer and the output projection of every layer replayed as one graph.
    x: [layers, B, S/N, C], y: [layers, B, S/N, N] (y[0] is computed once while sizing)."""

    def __init__(self, ctx: WorkerContext, x, w_qkv, heads: int, w_out, y, mesh: Mesh2D,
                 prologue: Optional[QKPrologue] = None, opts: Optional[CommOptions] = None,
                 layers: int = 1):
        opts = opts or CommOptions(check_finite=False)
        co = opts._c()
        pc = prologue._c() if prologue is not None else None
        _, b, s_, c = x.shape
        h = ctypes.c_void_p()
        self._keep = (x, w_qkv, w_out, y, prologue)
        self._ctx = ctx
        check(lib().fusp_graph_capture_block(
            ctx.handle, mesh.r, _ptr(x), _DT[x.dtype], b, s_, c, _ptr(w_qkv), heads,
            ctypes.byref(pc) if pc is not None else None, _ptr(w_out), int(w_out.shape[1]), _ptr(y),
            _DT[y.dtype], ctypes.byref(co), layers, x[0].numel() * x.element_size(),
            y[0].numel() * y.element_size(), _stream(), ctypes.byref(h)))
        self.handle = h

    def launch(self, stream=None):
        check(lib().fusp_graph_launch(self.handle, _stream(stream)))

    def close(self):
        if self.handle:
            lib().fusp_graph_destroy(self.handle)
            self.handle = None


class LayerGraph:
    """CUDA graph of `layers` back-to-back usp_attention calls (fusp_graph_capture_usp)."""

    def __init__(self, ctx: WorkerContext, q, k, v, out, mesh: Mesh2D,
                 opts: Optional[CommOptions] = None, layers: int = 1):
        opts = opts or CommOptions(check_finite=False)
        co = opts._c()
        # q/k/v/out: [layers, B, H, S, D]
        per_in = q[0].numel() * q.element_size()
        per_out = out[0].numel() * out.element_size()
        h = ctypes.c_void_p()
        self._keep = (q, k, v, out)
        self._ctx = ctx  # the graph replays the context's communicators: keep it alive
        check(lib().fusp_graph_capture_usp(ctx.handle, mesh.r, _ptr(q), _ptr(k), _ptr(v),
                                           _DT[q.dtype], _shape4(q[0]), _ptr(out),
                                           ctypes.byref(co), layers, per_in, per_out, _stream(),
                                           ctypes.byref(h)))
        self.handle = h

    def launch(self, stream=None):
        check(lib().fusp_graph_launch(self.handle, _stream(stream)))

    def close(self):
        if self.handle:
            lib().fusp_graph_destroy(self.handle)
            self.handle = None

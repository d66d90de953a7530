"""fastusp for B200: the FastUSP (arXiv 2602.10940) USP joint-attention layer.

Host-side mirror of the reference's uspsim API over the C ABI in
include/fastusp.h (libfastusp.so: hand-written sm_100a kernels + NCCL).
"""
from ._lib import (BF16, E4M3, F16, F32, DeadlockError, FabricError, FuspError, InvalidArgument, MeshError,
                   ShapeError, build)
from .api import (AttnResult, BlockGraph, CommOptions, Fabric, LayerGraph, Mesh2D, ProcessGroup,
                  QKPrologue, QuantizedTensor, rope_tables, RunReport, WorkerContext, attention_reference,
                  attention_schedule, attention_with_lse, build_mesh, decode_e4m3, dequantize, dequantize_blocks,
                  encode_e4m3, quantize_blocks, requantize,
                  gather_output, kernel_launch_count, make_mesh, merge_lse, quantize,
                  ring_attention_pipelined, ring_attention_serial, run_protocol, split_sequence,
                  ulysses_attention, usp_attention, usp_attention_host, out_projection,
                  usp_attention_proj, usp_block, usp_attention_with_lse, Resharded, detail, stage_f16, kFp8Max, kFp8MaxCode,
                  kFp8NanCode, peer_window_bytes)

__all__ = [n for n in dir() if not n.startswith("_")]

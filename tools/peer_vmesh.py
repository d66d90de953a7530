"""Peer-memory transport vs the in-process fabric on a virtual mesh (N ranks as threads on
cuda:0): wall time per FLUX-shaped layer (S = 4608, H = 24, U = N, R = 1), median of 3 runs of
10 layers after warm-up.  All ranks share one GPU, so the numbers are the N ranks' work
serialised on one device -- they show the transport's cost (fabric: a host rendezvous and
copy-engine pulls per all-to-all; peer: the pack / epilogue stores plus two 1-warp signal
kernels), not NVLink.  usage: CUDA_DEVICE_MAX_CONNECTIONS=32 python tools/peer_vmesh.py"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch  # noqa: E402

import paper_2602_10940_b200 as fu  # noqa: E402

h, s, d = 24, 4608, 128
g = torch.Generator(device="cuda")
g.manual_seed(1)
full = [torch.empty(1, h, s, d, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1, generator=g) for _ in range(3)]
for n in (2, 4, 8):
    sl = s // n
    shards = [[t[:, :, i * sl:(i + 1) * sl].contiguous() for i in range(n)] for t in full]
    mesh = fu.make_mesh(n, 1)
    row = {"n": n}
    for fp8 in (False, True):
        opts = fu.CommOptions(fp8_kv=fp8, check_finite=False, out_dtype=torch.float16)
        wb = fu.peer_window_bytes(n, 1, (1, h, sl, d), torch.bfloat16, opts)
        for peer in (False, True):
            def prog(ctx):
                if peer:
                    ctx.enable_peer_memory(wb)
                r = ctx.rank()
                args = (shards[0][r], shards[1][r], shards[2][r], mesh, opts)
                for _ in range(3):
                    fu.usp_attention(ctx, *args)
                ctx.synchronize()
                ts = []
                for _ in range(3):
                    t0 = time.perf_counter()
                    for _ in range(10):
                        fu.usp_attention(ctx, *args)
                    ctx.synchronize()
                    ts.append((time.perf_counter() - t0) / 10 * 1e6)
                return statistics.median(ts), ctx.peer_stats() if peer else None
            rep = fu.run_protocol(n, prog)
            us = max(x[0] for x in rep.results)
            row[f"{'fp8' if fp8 else 'bf16'}_{'peer' if peer else 'fabric'}_us_per_layer"] = round(us, 1)
    print(json.dumps(row), flush=True)

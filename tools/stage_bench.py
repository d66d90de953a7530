"""Interleaved A/B timing of the range-guarded staging kernel (fusp_stage_f16) across kernels.cu
variants (tools/build_variants_movers.sh), one process, CUDA events on the launching stream.
usage: python tools/stage_bench.py main VAR ...      ('main' = lib/libfastusp.so)
Prints one JSON line per (variant, dtype, cache state) with us and GB/s (algorithmic bytes:
read w_in + write 2 per element)."""
import ctypes
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2602_10940_b200")
DT = {torch.float32: 0, torch.float16: 1, torch.bfloat16: 2}


def load(name):
    path = os.path.join(PKG, "lib" if name == "main" else f"variants/{name}", "libfastusp.so")
    L = ctypes.CDLL(path, mode=os.RTLD_LOCAL)
    f = L.fusp_stage_f16
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                  ctypes.c_void_p, ctypes.c_void_p]
    return f


def main():
    names = sys.argv[1:] or ["main"]
    fns = {n: load(n) for n in names}
    heads, rows = int(os.environ.get("HEADS", 24)), int(os.environ.get("ROWS", 4608))
    flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
    s = torch.cuda.current_stream()
    res = {}
    for dt in (torch.bfloat16, torch.float32):
        x = torch.empty(heads, rows, 128, device="cuda", dtype=dt).uniform_(-1, 1)
        y = torch.empty(heads, rows, 128, device="cuda", dtype=torch.float16)
        e = torch.empty(heads, dtype=torch.int32, device="cuda")
        nbytes = x.numel() * (x.element_size() + 2)
        for rep in range(12):
            for n, f in fns.items():
                for cold in (False, True):
                    if cold:
                        flush.fill_(rep)
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    torch.cuda._sleep(200000)  # keep the GPU busy while the host enqueues: device time only
                    a.record(s)
                    rc = f(x.data_ptr(), DT[dt], heads, rows, y.data_ptr(), e.data_ptr(), s.cuda_stream)
                    b.record(s)
                    b.synchronize()
                    assert rc == 0, rc
                    if rep >= 2:
                        res.setdefault((n, str(dt), cold), []).append(a.elapsed_time(b) * 1e3)
            for cold in (False, True):  # reference mover: torch's own dtype-converting copy
                if cold:
                    flush.fill_(rep)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda._sleep(200000)
                a.record(s)
                y.copy_(x)
                b.record(s)
                b.synchronize()
                if rep >= 2:
                    res.setdefault(("torch_copy", str(dt), cold), []).append(a.elapsed_time(b) * 1e3)
        torch.cuda.synchronize()
        ok = torch.equal(y.float(), x.float().half().float()) and int(e.abs().sum()) == 0
        print(json.dumps({"dtype": str(dt), "last_variant_exact": bool(ok)}), flush=True)
    for (n, dt, cold), v in res.items():
        us = statistics.median(v)
        w = 4 if "float32" in dt else 2
        gbs = heads * rows * 128 * (w + 2) / (us * 1e-6) / 1e9
        print(json.dumps({"variant": n, "dtype": dt, "cold": cold, "us": round(us, 2),
                          "GBps": round(gbs, 1)}), flush=True)


if __name__ == "__main__":
    main()

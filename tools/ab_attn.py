"""Interleaved A/B timing of attention-kernel variants in ONE process (each variant .so loaded
with RTLD_LOCAL), so clock/thermal drift hits every variant alike.
usage: python tools/ab_attn.py VAR[:mode[:max_ctas]] ...   (VAR 'main' = lib/libfastusp.so)"""
import ctypes, json, os, statistics, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
import torch

PKG = os.path.join(ROOT, "paper_2602_10940_b200")
SHAPES = [("flux_u1", 24, 4608), ("flux_u2", 12, 4608), ("flux_u4", 6, 4608), ("flux_u8", 3, 4608),
          ("ring_u2r4_step", 12, 4224), ("qwen_u4r2_step", 6, 3584), ("qwen_u1", 24, 7168)]
if os.environ.get("SHAPES"):
    keep = os.environ["SHAPES"].split(",")
    SHAPES = [s for s in SHAPES if s[0] in keep]


class Shape4(ctypes.Structure):
    _fields_ = [("b", ctypes.c_int64), ("h", ctypes.c_int64), ("s", ctypes.c_int64), ("d", ctypes.c_int64)]


def load(spec):
    name, _, rest = spec.partition(":")
    mode, _, ctas = rest.partition(":")
    ctas = int(ctas) if ctas else 0
    path = os.path.join(PKG, "lib" if name == "main" else f"variants/{name}", "libfastusp.so")
    L = ctypes.CDLL(path)
    f = L.fusp_attention_with_lse_ex
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 2 + [Shape4, ctypes.c_int64, ctypes.c_void_p,
                                                                ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    if hasattr(L, "fusp_attention_schedule"):
        L.fusp_attention_schedule.argtypes = [ctypes.c_int, ctypes.c_int]
        L.fusp_attention_schedule(int({"whole": 1, "split": 2, "aligned": 3, "kv2": 4, "kv2split": 5}.get(mode, 0)), ctas)
    mode_id = int({"whole": 1, "split": 2, "aligned": 3, "kv2": 4, "kv2split": 5}.get(mode, 0))
    sched = getattr(L, "fusp_attention_schedule", None)

    def fn(*a):  # the schedule knob is process-global per library: set it before every call
        if sched is not None:
            sched(mode_id, ctas)
        return f(*a)
    return spec, fn


variants = [load(s) for s in sys.argv[1:]]
BF16, F16 = 2, 1
VDT = BF16 if os.environ.get("VDT") == "bf16" else F16  # V dtype handed to the kernel
for name, hp, s in SHAPES:
    q = torch.empty(1, hp, s, 128, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1)
    k = torch.empty_like(q).uniform_(-1, 1)
    v = torch.empty(1, hp, s, 128, device="cuda",
                    dtype=torch.bfloat16 if VDT == BF16 else torch.float16).uniform_(-1, 1)
    out = torch.empty(1, hp, s, 128, device="cuda", dtype=torch.float16)
    lse = torch.empty(1, hp, s, device="cuda", dtype=torch.float32)
    st = torch.cuda.current_stream().cuda_stream
    shp = Shape4(1, hp, s, 128)
    times = {sp: [] for sp, _ in variants}
    for rnd in range(6):
        for sp, f in variants:
            call = lambda: f(q.data_ptr(), k.data_ptr(), v.data_ptr(), BF16, VDT, shp, s, out.data_ptr(),
                             F16, lse.data_ptr(), st)
            for _ in range(2):
                assert call() == 0
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                call()
            e1.record(); e1.synchronize()
            if rnd > 0:
                times[sp].append(e0.elapsed_time(e1) * 100.0)
    fl = 4.0 * hp * s * s * 128
    print(json.dumps({"config": name, **{sp: {"us": round(statistics.median(t), 1),
                                               "tflops": round(fl / statistics.median(t) / 1e6, 1)}
                                          for sp, t in times.items()}}), flush=True)

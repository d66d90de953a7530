"""PCIe copy bandwidth on the GPU box: single H2D / D2H, H2D and D2H at once (duplex), and
H2D split over 1-4 streams.  Explains the e2e leg of bench.py (pinned host memory)."""
import torch

MB = 85


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


h = torch.empty(MB << 20, dtype=torch.uint8).pin_memory()
d = torch.empty_like(h, device="cuda")
h2 = torch.empty(28 << 20, dtype=torch.uint8).pin_memory()
d2 = torch.empty_like(h2, device="cuda")
n = MB << 20
print("h2d", MB, "MB", round(n / timed(lambda: d.copy_(h, non_blocking=True)) / 1e9, 1), "GB/s")
print("d2h", MB, "MB", round(n / timed(lambda: h.copy_(d, non_blocking=True)) / 1e9, 1), "GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def duplex():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t = timed(duplex)
print("duplex h2d 85 MB + d2h 28 MB", round(t * 1e6, 1), "us ->", round(n / t / 1e9, 1), "GB/s h2d-equivalent")
for ns in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(ns)]
    part = n // ns

    def multi():
        cur = torch.cuda.current_stream()
        for i, st in enumerate(ss):
            st.wait_stream(cur)
            with torch.cuda.stream(st):
                d[i * part:(i + 1) * part].copy_(h[i * part:(i + 1) * part], non_blocking=True)
        for st in ss:
            cur.wait_stream(st)

    print(f"h2d over {ns} streams", round(n / timed(multi) / 1e9, 1), "GB/s")

import torch, time
for mb in (28, 85):
    h = torch.empty(mb << 20, dtype=torch.uint8).pin_memory(); d = torch.empty_like(h, device="cuda")
    for direction in ("h2d", "d2h"):
        for _ in range(3):
            (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True)); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
        e1.record(); e1.synchronize()
        print(direction, mb, "MB", round(5 * (mb << 20) / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1), "GB/s")

"""Pinned host -> device copy bandwidth on the box (what bounds sage2_attn_host's e2e number):
one stream vs two streams, 3.2 GB total (C2-32K's q, k, v)."""
import torch
n = 3 * 4 * 32 * 32768 * 128 * 2
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for streams in (1, 2, 3):
    ss = [torch.cuda.Stream() for _ in range(streams)]
    part = n // streams
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i, s in enumerate(ss):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                d[i * part:(i + 1) * part].copy_(h[i * part:(i + 1) * part], non_blocking=True)
        for s in ss:
            e1.wait_stream(s) if hasattr(e1, "wait_stream") else None
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
    print(f"{streams} stream(s): H2D {n / e0.elapsed_time(e1) / 1e6:.1f} GB/s")
o = torch.empty(n // 3, dtype=torch.uint8).pin_memory()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); o.copy_(d[: n // 3], non_blocking=True); e1.record(); torch.cuda.synchronize()
print(f"D2H {n / 3 / e0.elapsed_time(e1) / 1e6:.1f} GB/s")

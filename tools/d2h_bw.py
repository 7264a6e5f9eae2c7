"""D2H bandwidth into pinned host memory with 1..4 streams (copy engines)."""
import torch
n = 192 * 1024 * 1024
src = torch.empty(n, dtype=torch.uint8, device="cuda")
for ns in (1, 2, 3, 4):
    dst = [torch.empty(n // ns, dtype=torch.uint8, pin_memory=True) for _ in range(ns)]
    streams = [torch.cuda.Stream() for _ in range(ns)]
    for rep in range(2):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for i, s in enumerate(streams):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                dst[i].copy_(src[i * (n // ns):(i + 1) * (n // ns)], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{ns} streams: {n / ms / 1e6:.1f} GB/s")
# H2D for reference
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); src.copy_(h, non_blocking=True); e1.record(); torch.cuda.synchronize()
print(f"H2D 1 stream: {n / e0.elapsed_time(e1) / 1e6:.1f} GB/s")

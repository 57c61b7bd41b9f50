"""Dev probe: back-to-back pinned host -> device copy rate by copy size and stream count."""
import torch

MB = 1 << 20
src = torch.empty(16 * MB, dtype=torch.uint8, pin_memory=True)
dst = torch.empty(16 * MB, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(2)]


def run(size, nstreams, reps=200):
    total = 0
    for _ in range(10):
        dst[:size].copy_(src[:size], non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in streams[:nstreams]:
        s.wait_event(e0)
    for i in range(reps):
        s = streams[i % nstreams]
        with torch.cuda.stream(s):
            dst[(i % 2) * 8 * MB:(i % 2) * 8 * MB + size].copy_(src[:size], non_blocking=True)
        total += size
    for s in streams[:nstreams]:
        e1.wait_stream(s) if hasattr(e1, "wait_stream") else None
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    return total / ms / 1e6


for size in (1250000, 2500000, 5000000):
    for ns in (1, 2):
        print(f"{size / 1e6:5.2f} MB x{ns} streams: {run(size, ns):6.1f} GB/s")

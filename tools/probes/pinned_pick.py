"""Dev probe: H2D rate of several simultaneously-live pinned buffers in one process
(is the slow / fast H2D mode a property of the buffer or of the process?)."""
import torch

n = 1_250_000
dst = torch.empty(n, dtype=torch.uint8, device="cuda")
bufs = [torch.empty(n + k * 4096, dtype=torch.uint8, pin_memory=True) for k in range(8)]
big = torch.empty(64 << 20, dtype=torch.uint8, pin_memory=True)
bufs.append(big[:n])
bufs.append(big[32 << 20:(32 << 20) + n])
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
out = []
for b in bufs:
    b.fill_(1)
    for _ in range(3):
        dst.copy_(b[:n], non_blocking=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        dst.copy_(b[:n], non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    out.append(20 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9)
print(" ".join(f"{x:5.1f}" for x in out), "GB/s")

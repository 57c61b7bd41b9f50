import torch, time
n, cases = 5, 1_000_000
pitch = (cases + 31) // 32 * 32
a = torch.empty((n, cases), dtype=torch.int8, pin_memory=True)
da = torch.empty((n, pitch), dtype=torch.int8, device="cuda")
b = torch.empty((n, pitch // 2), dtype=torch.uint8, pin_memory=True)
db = torch.empty((n, pitch // 2), dtype=torch.uint8, device="cuda")
print("pinned", a.is_pinned(), b.is_pinned())
for name, fn in [("int8 2D 5MB", lambda: da[:, :cases].copy_(a, non_blocking=True)),
                 ("u8 contiguous 2.5MB", lambda: db.copy_(b, non_blocking=True))]:
    for _ in range(5): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): fn()
    e1.record(); torch.cuda.synchronize()
    print(name, e0.elapsed_time(e1) / 50 * 1e3, "us")

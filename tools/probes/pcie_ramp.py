"""Dev probe: H2D rate trajectory after a period of device-only work, with the NVML PCIe
link generation / width (does the link come back up under sustained uploads?)."""
import time

import pynvml
import torch

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)


def link():
    return (pynvml.nvmlDeviceGetCurrPcieLinkGeneration(h), pynvml.nvmlDeviceGetCurrPcieLinkWidth(h),
            pynvml.nvmlDeviceGetMaxPcieLinkGeneration(h))


n = 1_250_000
host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
host.fill_(1)
dst = torch.empty(n, dtype=torch.uint8, device="cuda")
a = torch.randn(8192, 8192, device="cuda")
print("idle link", link())
t0 = time.perf_counter()
while time.perf_counter() - t0 < 2.0:  # device-only work, no PCIe traffic
    for _ in range(10):
        a = a @ a
        a = a / a.norm()
    torch.cuda.synchronize()
print("after compute link", link())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
traj = []
while time.perf_counter() - t0 < 2.0:
    e0.record()
    for _ in range(8):
        dst.copy_(host, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    traj.append((time.perf_counter() - t0, 8 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9))
    if len(traj) in (1, 50, 400):
        print(f"  t={traj[-1][0] * 1e3:7.1f} ms rate {traj[-1][1]:5.1f} GB/s link {link()}")
for ms in (10, 25, 50, 100, 200, 500, 1000, 1900):
    r = [x for t, x in traj if t * 1e3 <= ms]
    print(f"  by {ms:5d} ms: last {r[-1]:5.1f} GB/s")

"""Dev tool: H2D bandwidth of pinned buffers by allocation method (torch pinned vs
2 MB-aligned THP mmap + cudaHostRegister), repeated to expose run-to-run variance."""
import ctypes, mmap, os, sys
import numpy as np
import torch

print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(),
      open("/sys/kernel/mm/transparent_hugepage/defrag").read().strip())
cudart = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
nbytes = 2_500_000
dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda")


def bw(host):
    for _ in range(5):
        dst.copy_(host, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(40):
        dst.copy_(host, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 40 * 1e3


for trial in range(4):
    t = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    t.fill_(1)
    print(f"torch pinned      {bw(t):6.1f} us")
    size = 4 << 20
    buf = mmap.mmap(-1, size + (2 << 20), flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    addr = ctypes.addressof(ctypes.c_char.from_buffer(buf))
    al = (addr + (2 << 20) - 1) & ~((2 << 20) - 1)
    libc = ctypes.CDLL("libc.so.6")
    libc.madvise(ctypes.c_void_p(al), ctypes.c_size_t(size), 14)  # MADV_HUGEPAGE
    arr = np.frombuffer((ctypes.c_char * size).from_address(al), dtype=np.uint8)
    arr[:] = 1
    rc = torch.cuda.cudart().cudaHostRegister(al, size, 0)
    h = torch.from_numpy(arr[:nbytes])
    print(f"THP + register    {bw(h):6.1f} us  (register rc={rc}, pinned={h.is_pinned()})")
    torch.cuda.cudart().cudaHostUnregister(al)

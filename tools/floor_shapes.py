"""Event-timed empty kernels of several launch shapes after an sg_flush_l2 (dev probe)."""
import ctypes
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1511_06416_b200 import _lib  # noqa: E402

_lib.load()
s = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
big = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rd = torch.ones(32 << 20, dtype=torch.int64, device="cuda")
ev = []
for _ in range(2):
    h = ctypes.c_uint64()
    _lib.call("sg_event_create", ctypes.byref(h))
    ev.append(h.value)
for ctas, thr, sm in [(147, 1024, 120 * 1024), (147, 1024, 0), (147, 512, 120 * 1024), (148, 256, 0), (1, 32, 0),
                      (147, 1024, 200 * 1024)]:
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        _lib.call("sg_event_record", ev[0], s())
        _lib.call("sg_noop", ctas, thr, sm, s())
        _lib.call("sg_event_record", ev[1], s())
    for flush in (True, False):
        out = []
        for k in range(25):
            if flush:
                _lib.call("sg_flush_l2", big.data_ptr(), rd.data_ptr(), 256 << 20, k, s())
            g.replay()
            torch.cuda.synchronize()
            ms = ctypes.c_float()
            _lib.call("sg_event_elapsed", ev[0], ev[1], ctypes.byref(ms))
            if k >= 5:
                out.append(ms.value * 1e3)
        print(f"ctas {ctas:4d} threads {thr:5d} smem {sm // 1024:4d} KB flush {flush!s:5s}: "
              f"{statistics.mean(out):6.2f} us (min {min(out):.2f})", flush=True)

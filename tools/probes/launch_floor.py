"""Dev probe: events-around-an-empty-kernel time by launch shape, L2 flushed first."""
import ctypes
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch

from paper_1511_06416_b200 import _lib

_lib.load()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush_rd = torch.ones(32 << 20, dtype=torch.int64, device="cuda")
ev = []
for _ in range(2):
    h = ctypes.c_uint64()
    _lib.call("sg_event_create", ctypes.byref(h))
    ev.append(h.value)
for ctas, threads, smem in [(147, 1024, 120 << 10), (147, 1024, 0), (294, 512, 60 << 10), (147, 512, 120 << 10),
                            (147, 256, 0), (1, 32, 0), (147, 1024, 200 << 10)]:
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        s = torch.cuda.current_stream().cuda_stream
        _lib.call("sg_event_record", ev[0], s)
        _lib.call("sg_noop", ctas, threads, smem, s)
        _lib.call("sg_event_record", ev[1], s)
    out = []
    for k in range(15):
        for flushed in (True, False):
            if flushed:
                _lib.call("sg_flush_l2", flush.data_ptr(), flush_rd.data_ptr(), 256 << 20, k,
                          torch.cuda.current_stream().cuda_stream)
            g.replay()
            torch.cuda.synchronize()
            ms = ctypes.c_float()
            _lib.call("sg_event_elapsed", ev[0], ev[1], ctypes.byref(ms))
            if k >= 3:
                out.append((flushed, ms.value * 1e3))
    f = statistics.mean(x for fl, x in out if fl)
    w = statistics.mean(x for fl, x in out if not fl)
    print(f"{ctas:4d} x {threads:4d} thr, {smem >> 10:3d} KB smem: after flush {f:5.2f} us, warm {w:5.2f} us")

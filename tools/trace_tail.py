"""Dev tool: per-CTA timeline of the merged joint step tail (debug build -DSG_FINISH_TRACE).

  python paper_1511_06416_b200/_build.py -DSG_FINISH_TRACE --out=paper_1511_06416_b200/lib_variant_trace.so
  SAMEGIBBS_LIB=$PWD/paper_1511_06416_b200/lib_variant_trace.so python tools/trace_tail.py [cold]
"""
import ctypes
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_1511_06416_b200 as sg
from paper_1511_06416_b200 import _lib
from paper_1511_06416_b200.device import stream_handle
from paper_1511_06416_b200.engine import Engine
from paper_1511_06416_b200.io import bundled_network_path, load_network_file

lib = _lib.load()
lib.sg_debug_tail_trace.argtypes = [ctypes.c_void_p]
lib.sg_debug_tail_finish_trace.argtypes = [ctypes.c_void_p]
net, truth = load_network_file(bundled_network_path("koller"))
cases = 1_000_000
obs = sg.forward_sample_device(net, truth, cases, seed=1, hide_fraction=0.5, mask_seed=2)
cold = "cold" in sys.argv
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush_rd = torch.ones(32 << 20, dtype=torch.int64, device="cuda")
cfg = sg.SamplerConfig(same_m=10, minibatch_size=cases, seed=3, rng="joint")
eng = Engine(net, cfg)
mb = next(iter(sg.DeviceSource(obs, cases, cases)))
eng.visit(mb, 0, 10)
new = eng.prev_counts[0].clone()
f = eng.finish_args(new, eng.prev_counts[0], 12345)
G = 1 + 32 * 4
res = []
for k in range(20):
    if cold:
        flush.fill_(k & 0xFF)
        flush_rd.sum()
    eng.step_tail(f, stream_handle())
    torch.cuda.synchronize()
    t = (ctypes.c_ulonglong * 640)()
    lib.sg_debug_tail_trace(ctypes.cast(t, ctypes.c_void_p))
    ft = (ctypes.c_ulonglong * 8)()
    lib.sg_debug_tail_finish_trace(ctypes.cast(ft, ctypes.c_void_p))
    t0 = min(t[4 * b] for b in range(G))
    lead_start, lead_end = t[0] - t0, t[1] - t0
    starts = [t[4 * b] - t0 for b in range(1, G)]
    seen = [t[4 * b + 1] - t0 for b in range(1, G)]
    ends = [t[4 * b + 2] - t0 for b in range(1, G)]
    phases = [ft[i] - t0 for i in (7, 0, 1, 2, 3, 4, 5, 6)]
    res.append((lead_start, lead_end, max(starts), statistics.median(seen), max(ends), phases))
r = res[len(res) // 2]
print(("cold" if cold else "warm"), f"leader {r[0]/1e3:.2f}..{r[1]/1e3:.2f} us; slices start<= {r[2]/1e3:.2f}, "
      f"flag seen ~{r[3]/1e3:.2f}, last end {r[4]/1e3:.2f} us")
print("  finish phases (us from grid start):", " ".join(f"{x/1e3:.2f}" for x in r[5]))

"""Dev tool: phase timings of the single-CTA step tail (debug build with -DSG_FINISH_TRACE).

  python paper_1511_06416_b200/_build.py -DSG_FINISH_TRACE --out=build/lib_trace.so
  SAMEGIBBS_LIB=$PWD/build/lib_trace.so python tools/trace_finish.py
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
lib.sg_debug_finish_trace.argtypes = [ctypes.c_void_p]
net, truth = load_network_file(bundled_network_path("koller"))
cases = 1_000_000
obs = sg.forward_sample_device(net, truth, cases, seed=1, hide_fraction=0.5, mask_seed=2)
names = ["stage blobs", "wait + key", "accumulate + gamma", "rows (Dirichlet)", "tables", "small tables",
         "clear + keys"]
cold = "cold" in sys.argv
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush_rd = torch.ones(32 << 20, dtype=torch.int64, device="cuda")
rng = "joint" if "joint" in sys.argv else "fast"
for map_est in (False, True):
    cfg = sg.SamplerConfig(same_m=10, minibatch_size=cases, seed=3, rng=rng, map_estimate=map_est)
    eng = Engine(net, cfg)
    mb = next(iter(sg.DeviceSource(obs, cases, cases)))
    eng.visit(mb, 0, 10)
    new = eng.prev_counts[0].clone()
    f = eng.finish_args(new, eng.prev_counts[0], 12345)
    rows = []
    for k in range(30):
        if cold:
            flush.fill_(k & 0xFF)
            flush_rd.sum()
        _lib.call("sg_step_finish", eng.pack.ref, eng.small_ptr, f, stream_handle())
        torch.cuda.synchronize()
        t = (ctypes.c_ulonglong * 8)()
        lib.sg_debug_finish_trace(ctypes.cast(t, ctypes.c_void_p))
        order = [t[7], t[0], t[1], t[2], t[3], t[4], t[5], t[6]]
        rows.append([b - a for a, b in zip(order, order[1:])])
    med = [statistics.median(r[i] for r in rows[5:]) for i in range(7)]
    print(rng, "cold" if cold else "warm", "map" if map_est else "sampled", " | ".join(f"{n} {v / 1e3:.2f}" for n, v in zip(names, med)),
          f"| total {sum(med) / 1e3:.2f} us")

"""Dev tool: globaltimer timeline of graph-replayed joint steps (debug build
-DSG_FINISH_TRACE): sweep CTAs, the tail's CTA 0 phases, the row slices.

  python paper_1511_06416_b200/_build.py -DSG_FINISH_TRACE --out=paper_1511_06416_b200/lib_variant_trace.so
  SAMEGIBBS_LIB=$PWD/paper_1511_06416_b200/lib_variant_trace.so python tools/trace_step.py [cold]
"""
import ctypes
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_1511_06416_b200 as sg
from paper_1511_06416_b200 import _lib
from paper_1511_06416_b200.engine import Engine, StepGraphs
from paper_1511_06416_b200.io import bundled_network_path, load_network_file

lib = _lib.load()
for f in ("sg_debug_tail_trace", "sg_debug_tail_finish_trace", "sg_debug_sweep_trace"):
    getattr(lib, f).argtypes = [ctypes.c_void_p]
net, truth = load_network_file(bundled_network_path("koller"))
cases, m = 1_000_000, 10
obs = sg.forward_sample_device(net, truth, cases, seed=1, hide_fraction=0.5, mask_seed=2)
cold = "cold" in sys.argv
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush_rd = torch.ones(32 << 20, dtype=torch.int64, device="cuda")
cfg = sg.SamplerConfig(same_m=10, minibatch_size=cases, seed=3, rng="joint")
eng = Engine(net, cfg)
mb = next(iter(sg.DeviceSource(obs, cases, cases)))
for p in range(3):
    eng.visit(mb, p, 10)
g = StepGraphs(eng, mb, 10, range(3, 40))
rows = []
prev_end = None
for k in range(12):
    if cold:
        _lib.call("sg_flush_l2", flush.data_ptr(), flush_rd.data_ptr(), 256 << 20, k,
                  torch.cuda.current_stream().cuda_stream)
    if cold:
        torch.cuda.synchronize()
    g.step()
    if cold or k % 2 == 1:
        torch.cuda.synchronize()
    sw = (ctypes.c_ulonglong * 1280)()
    lib.sg_debug_sweep_trace(ctypes.cast(sw, ctypes.c_void_p))
    tt = (ctypes.c_ulonglong * (16 * 160 + 160))()
    lib.sg_debug_tail_trace(ctypes.cast(tt, ctypes.c_void_p))
    ft = (ctypes.c_ulonglong * 12)()
    lib.sg_debug_tail_finish_trace(ctypes.cast(ft, ctypes.c_void_p))
    nsw = 147
    t0 = min(sw[8 * b] for b in range(nsw))
    roles = [int(tt[16 * 160 + b]) for b in range(129)]
    c0 = roles.index(0)
    sl = [b for b in range(129) if roles[b] >= 1]
    T = lambda b, k: tt[16 * b + k]  # noqa: E731
    r = {
        "sweep first start": 0,
        "sweep last start": max(sw[8 * b] for b in range(nsw)) - t0,
        "sweep prologue issued (median)": statistics.median(sw[8 * b + 2] for b in range(nsw)) - t0,
        "sweep draws start (median)": statistics.median(sw[8 * b + 3] for b in range(nsw)) - t0,
        "sweep draws start (last)": max(sw[8 * b + 3] for b in range(nsw)) - t0,
        "sweep first end": min(sw[8 * b + 1] for b in range(nsw)) - t0,
        "sweep last end": max(sw[8 * b + 1] for b in range(nsw)) - t0,
        "tail CTA0 start": T(c0, 0) - t0,
        "tail: early inputs done": ft[0] - t0,
        "tail: wait+key": ft[1] - t0,
        "tail: counts loaded": ft[8] - t0,
        "tail: gamma drawn": ft[9] - t0,
        "tail: acc+gamma": ft[2] - t0,
        "tail: rows": ft[3] - t0,
        "tail: tables": ft[4] - t0,
        "tail: clear+keys": ft[6] - t0,
        "tail CTA0 end": T(c0, 1) - t0,
        "slices entry (median)": statistics.median(T(b, 10) for b in sl) - t0,
        "slices ticket (median)": statistics.median(T(b, 0) for b in sl) - t0,
        "slices last start": max(T(b, 0) for b in sl) - t0,
        "slices blobs staged + share checked (median)": statistics.median(T(b, 8) for b in sl) - t0,
        "slices part 1 done (median)": statistics.median(T(b, 9) for b in sl) - t0,
        "slices prep done (median)": statistics.median(T(b, 7) for b in sl) - t0,
        "slices prep done (last)": max(T(b, 7) for b in sl) - t0,
        "slices flag seen (median)": statistics.median(T(b, 1) for b in sl) - t0,
        "slices conditionals done (median)": statistics.median(T(b, 3) for b in sl) - t0,
        "slices rows loop start (median)": statistics.median(T(b, 4) for b in sl) - t0,
        "slices gammas loaded (median)": statistics.median(T(b, 5) for b in sl) - t0,
        "slices Dirichlet rows (median)": statistics.median(T(b, 6) for b in sl) - t0,
        "slices median end": statistics.median(T(b, 2) for b in sl) - t0,
        "slices last end": max(T(b, 2) for b in sl) - t0,
        "slowest slice role": float(roles[max(sl, key=lambda b: T(b, 2))]),
        "slowest: start": T(max(sl, key=lambda b: T(b, 2)), 0) - t0,
        "slowest: prep done": T(max(sl, key=lambda b: T(b, 2)), 7) - t0,
        "slowest: flag seen": T(max(sl, key=lambda b: T(b, 2)), 1) - t0,
        "slowest: cond done": T(max(sl, key=lambda b: T(b, 2)), 3) - t0,
        "slowest: rows start": T(max(sl, key=lambda b: T(b, 2)), 4) - t0,
        "slowest: gammas loaded": T(max(sl, key=lambda b: T(b, 2)), 5) - t0,
        "slowest: Dirichlet rows": T(max(sl, key=lambda b: T(b, 2)), 6) - t0,
    }
    r["gap: prev tail end -> sweep start"] = (t0 - prev_end) if (prev_end and not cold) else 0
    prev_end = max(T(b, 2) for b in sl)
    rows.append(r)
print("cold" if cold else "warm", "(us from the first sweep CTA's start, median of steps 2..11)")
for key in rows[0]:
    v = statistics.median(r[key] for r in rows[2:])
    print(f"  {key:34s} {v / 1e3 if 'role' not in key else v:8.2f}")

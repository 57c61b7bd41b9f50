"""Dev tool: per-launch GPU time of one minibatch step (eager visits, events
between launches), with the L2 flushed before each step (bench.py's rule) or
warm.   python tools/step_breakdown.py [joint|fast] [cold|warm]
"""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_1511_06416_b200 as sg
from paper_1511_06416_b200 import _lib
from paper_1511_06416_b200.engine import Engine
from paper_1511_06416_b200.io import bundled_network_path, load_network_file

rng = sys.argv[1] if len(sys.argv) > 1 else "joint"
cold = (sys.argv[2] if len(sys.argv) > 2 else "cold") == "cold"
net, truth = load_network_file(bundled_network_path("koller"))
cases, m = 1_000_000, 10
obs = sg.forward_sample_device(net, truth, cases, seed=1, hide_fraction=0.5, mask_seed=2)
cfg = sg.SamplerConfig(same_m=m, minibatch_size=cases, seed=3, rng=rng)
eng = Engine(net, cfg)
mb = next(iter(sg.DeviceSource(obs, cases, cases)))
for p in range(3):
    eng.visit(mb, p, m)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush_rd = torch.ones(32 << 20, dtype=torch.int64, device="cuda")
marks = []
orig = _lib.call


def call(name, *args):
    orig(name, *args)
    if marks is not None:
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        marks.append((name, e))


_lib.call = call
rows = {}
for k in range(30):
    if cold:
        flush.fill_(k & 0xFF)
        flush_rd.sum()
    marks = []
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.visit(mb, 3 + k, m)
    torch.cuda.synchronize()
    prev = e0
    for name, e in marks:
        rows.setdefault(name, []).append(prev.elapsed_time(e) * 1e3)
        prev = e
    rows.setdefault("total", []).append(e0.elapsed_time(prev) * 1e3)
marks = None
print(f"{rng} {'cold' if cold else 'warm'} (median us over 25 steps):")
for name, v in rows.items():
    print(f"  {name:20s} {statistics.median(v[5:]):8.2f}")

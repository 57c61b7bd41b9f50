"""Dev probe: back-to-back C2 visits replayed one per graph vs two per graph."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch

import paper_1511_06416_b200 as sg
from paper_1511_06416_b200.engine import Engine, StepGraphs
from paper_1511_06416_b200.io import bundled_network_path, load_network_file

net, truth = load_network_file(bundled_network_path("koller"))
cases, m = 1_000_000, 10
obs = sg.forward_sample_device(net, truth, cases, seed=1, hide_fraction=0.5, mask_seed=2)
mb = next(iter(sg.DeviceSource(obs, cases, cases)))
cfg = sg.SamplerConfig(same_m=m, minibatch_size=cases, num_passes=1, seed=300, rng="joint")
eng = Engine(net, cfg)
for w in range(3):
    eng.visit(mb, w, m)
g = StepGraphs(eng, mb, m, range(3, 3 + 2000), obs_bits=2)


def timed(fn, n):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


print("one visit per graph:", round(timed(g.step, 200), 1), "us/visit")
g2 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g2):
    g._record(0)
    g._record(1)
print("two visits per graph:", round(timed(g2.replay, 100) / 2, 1), "us/visit")
g4 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g4):
    for k in range(4):
        g._record(k)
print("four visits per graph:", round(timed(g4.replay, 50) / 4, 1), "us/visit")

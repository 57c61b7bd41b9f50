"""Dev tool: per-step timeline (copy stream vs replay) of StepGraphs.step(host_mb)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_1511_06416_b200 as sg
from paper_1511_06416_b200.engine import Engine, StepGraphs
from paper_1511_06416_b200.io import bundled_network_path, load_network_file, pack_nibbles

nib = "int8" not in sys.argv
net, truth = load_network_file(bundled_network_path("koller"))
cases, m = 1_000_000, 10
obs = sg.forward_sample_device(net, truth, cases, seed=1, hide_fraction=0.5, mask_seed=2)
mb = next(iter(sg.DeviceSource(obs, cases, cases)))
cfg = sg.SamplerConfig(same_m=m, minibatch_size=cases, num_passes=1, seed=300, rng="joint")
eng = Engine(net, cfg)
for w in range(3):
    eng.visit(mb, w, m)
g = StepGraphs(eng, mb, m, range(3, 200), nibbles=nib)
if nib:
    p4 = g.obs_bufs[0].shape[1] * 2
    host = torch.empty((5, p4 // 2), dtype=torch.uint8, pin_memory=True)
    host.copy_(pack_nibbles(obs[:, :cases], p4).cpu())
else:
    host = torch.empty((5, cases), dtype=torch.int8, pin_memory=True)
    host.copy_(obs[:, :cases])
hmb = sg.Minibatch(index=0, values=host, weights=np.ones(cases), num_real=cases)
# instrument: events around the upload (copy stream) and the replay (main stream)
marks = []
orig_replays = [gr.replay for gr in g.graphs]
for i, gr in enumerate(g.graphs):
    def rep(orig=orig_replays[i]):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); orig(); b.record()
        marks.append(("replay", a, b))
    gr.replay = rep
t0 = torch.cuda.Event(enable_timing=True)
for _ in range(3):
    g.step(hmb)
torch.cuda.synchronize()
marks.clear()
cs = g._copy_stream
t0.record()
for k in range(6):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(cs)
    g.step(hmb)
    b.record(cs)
    marks.append(("copy", a, b))
torch.cuda.synchronize()
for name, a, b in marks:
    print(f"{name:7s} {t0.elapsed_time(a) * 1e3:8.1f} -> {t0.elapsed_time(b) * 1e3:8.1f} us")

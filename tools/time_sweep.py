"""Dev tool: mean event time of the joint sweep launch (eager visits, L2 flushed), for A/B variants."""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_1511_06416_b200 as sg
from paper_1511_06416_b200.engine import Engine
from paper_1511_06416_b200.io import bundled_network_path, load_network_file

net, truth = load_network_file(bundled_network_path("koller"))
cases = 1_000_000
obs = sg.forward_sample_device(net, truth, cases, seed=1, hide_fraction=0.5, mask_seed=2)
cfg = sg.SamplerConfig(same_m=10, minibatch_size=cases, seed=3, rng="joint")
eng = Engine(net, cfg)
mb = next(iter(sg.DeviceSource(obs, cases, cases)))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
eng.visit(mb, 0, 10)
eng.sweep_events = []
for k in range(25):
    flush.fill_(k & 0xFF)
    if "sleep" in sys.argv:
        torch.cuda._sleep(200_000)
    eng.visit(mb, 1 + k, 10)
torch.cuda.synchronize()
t = [a.elapsed_time(b) * 1e3 for a, b, _ in eng.sweep_events[5:]]
print(f"sweep {statistics.mean(t):.1f} us (min {min(t):.1f})")

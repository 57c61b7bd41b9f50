"""Debug: eager vs graph runs of single cases (run each in its own process)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1511_06416_b200 as sg  # noqa: E402
from paper_1511_06416_b200.io import bundled_network_path, load_network_file  # noqa: E402

net, truth = load_network_file(bundled_network_path("koller"))
case = int(sys.argv[1])
CASES = [
    dict(rng="fast", same_m=2, map_estimate=True, sweeps_per_minibatch=2),
    dict(rng="joint", same_m=10),
    dict(rng="fast", same_m=2, map_estimate=True, sweeps_per_minibatch=1),
    dict(rng="fast", same_m=2, map_estimate=False, sweeps_per_minibatch=2),
    dict(rng="joint", same_m=10, num_passes=2),
]
kw = dict(CASES[case])
passes = kw.pop("num_passes", 6)
mbs = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
cases = 5000
obs = sg.forward_sample_device(net, truth, cases, seed=5, hide_fraction=0.5, mask_seed=6)
cfg = sg.SamplerConfig(minibatch_size=mbs, num_passes=passes, seed=9, **kw)
res = []
for graphs in (False, True):
    def hook(e):
        e.graph_replay = graphs
    cpts, tr = sg.run(net, sg.DeviceSource(obs, cases, mbs), cfg, truth=truth, engine_hook=hook)
    torch.cuda.synchronize()
    res.append(cpts)
    print("graphs", graphs, [round(r.kl_avg, 6) for r in tr.records], flush=True)
print("equal:", all(np.array_equal(a, b) for a, b in zip(res[0].tables, res[1].tables)))

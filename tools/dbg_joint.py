"""Debug: eager joint visits over several minibatches, synchronising after each."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1511_06416_b200 as sg  # noqa: E402
from paper_1511_06416_b200.engine import Engine  # noqa: E402
from paper_1511_06416_b200.io import bundled_network_path, load_network_file  # noqa: E402

net, truth = load_network_file(bundled_network_path("koller"))
cases, mbs, m, rng = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
obs = sg.forward_sample_device(net, truth, cases, seed=5, hide_fraction=0.5, mask_seed=6)
cfg = sg.SamplerConfig(minibatch_size=mbs, num_passes=6, seed=9, same_m=m, rng=rng)
eng = Engine(net, cfg)
src = sg.DeviceSource(obs, cases, mbs)
for p in range(6):
    for mb in src:
        try:
            eng.visit(mb, p, m)
            torch.cuda.synchronize()
        except Exception as e:  # noqa: BLE001
            print(f"FAILED pass {p} mb {mb.index} size {mb.size} real {mb.num_real}: {e}", flush=True)
            raise SystemExit(1)
    print(f"pass {p} ok err={eng.err.read()}", flush=True)

"""Dev probe: sg_small_prepare on a C2 minibatch, repeated (for ncu)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch

import paper_1511_06416_b200 as sg
from paper_1511_06416_b200 import _lib
from paper_1511_06416_b200.engine import SmallBatch, Engine
from paper_1511_06416_b200.io import bundled_network_path, load_network_file

net, truth = load_network_file(bundled_network_path("koller"))
B = 1_000_000
obs = sg.forward_sample_device(net, truth, B, seed=100, hide_fraction=0.5, mask_seed=200)
cfg = sg.SamplerConfig(same_m=10, minibatch_size=B, seed=300, rng="joint", accumulator_mode="exponential")
eng = Engine(net, cfg)
db = SmallBatch(net.num_vars, 10, B, torch.device("cuda"))
key = torch.zeros(1, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 10):
    _lib.call("sg_small_prepare", eng.pack.small_ref, obs.data_ptr(), obs.stride(0), B, 10, 0, 0, 1,
              db.scratch.data_ptr(), db.pattern.data_ptr(), db.case_id.data_ptr(), db.lanes.data_ptr(), db.lane_ld,
              key.data_ptr(), s)
torch.cuda.synchronize()
print("ok")

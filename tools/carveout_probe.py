"""Dev tool: does the L1/shared carveout switch after the L2-flush kernels cost the step / sweep time?
Replays timed step graphs (external events around the sweep node) after a torch L2 flush, with and
without an empty max-shared kernel (sg_noop, the sweep's launch shape) between the flush and the step."""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_1511_06416_b200 as sg
from paper_1511_06416_b200 import _lib
from paper_1511_06416_b200.engine import Engine, StepGraphs
from paper_1511_06416_b200.io import bundled_network_path, load_network_file

net, truth = load_network_file(bundled_network_path("koller"))
cases = 1_000_000
obs = sg.forward_sample_device(net, truth, cases, seed=1, hide_fraction=0.5, mask_seed=2)
cfg = sg.SamplerConfig(same_m=10, minibatch_size=cases, seed=3, rng="joint")
eng = Engine(net, cfg)
mb = next(iter(sg.DeviceSource(obs, cases, cases)))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush_rd = torch.ones(32 << 20, dtype=torch.int64, device="cuda")
for w in range(3):
    eng.visit(mb, w, 10)
torch.cuda.synchronize()
sms = torch.cuda.get_device_properties(0).multi_processor_count
base = 10
for prime in (False, True, False, True):
    tg = StepGraphs(eng, mb, 10, range(base, base + 30), obs_bits=2, timing=True)
    base += 40
    sw, st = [], []
    for k in range(30):
        flush.fill_(k & 0xFF)
        flush_rd.sum()
        if prime:
            _lib.call("sg_noop", sms, 1024, 120 * 1024, torch.cuda.current_stream().cuda_stream)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        tg.step()
        b.record()
        torch.cuda.synchronize()
        if k >= 3:
            sw.append(tg.sweep_ms() * 1e3)
            st.append(a.elapsed_time(b) * 1e3)
    tg.finish()
    print(f"prime={prime}: sweep {statistics.mean(sw):.1f} us  step {statistics.mean(st):.1f} us")

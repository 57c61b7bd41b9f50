"""Dev tool: does the L1/shared carveout switch after the L2-flush kernels cost the sweep time?
Times the joint sweep (eager events, L2 flushed) with and without a tiny max-shared kernel
launched between the flush and the visit."""
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

net, truth = load_network_file(bundled_network_path("koller"))
cases = 1_000_000
obs = sg.forward_sample_device(net, truth, cases, seed=1, hide_fraction=0.5, mask_seed=2)
cfg = sg.SamplerConfig(same_m=10, minibatch_size=cases, seed=3, rng="joint")
eng = Engine(net, cfg)
mb = next(iter(sg.DeviceSource(obs, cases, cases)))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
eng.visit(mb, 0, 10)
for prime in (False, True, False, True):
    eng.sweep_events = []
    for k in range(20):
        flush.fill_(k & 0xFF)
        if prime:  # the step tail kernel (max-shared carveout) on a dummy sync pair: re-primes the SMs' carveout
            _lib.call("sg_copy_small", eng.vprob.data_ptr(), eng.vprob.data_ptr(), 8, stream_handle())
        torch.cuda._sleep(100_000)
        eng.visit(mb, 1 + k + (100 if prime else 0), 10)
    torch.cuda.synchronize()
    t = [a.elapsed_time(b) * 1e3 for a, b, _ in eng.sweep_events[3:]]
    print(f"prime={prime}: sweep {statistics.mean(t):.1f} us")

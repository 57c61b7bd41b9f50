"""Dev tool: e2e step time of host-fed step graphs (in-graph upload of the
next block, CPT read-back) vs plain replays."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_1511_06416_b200 as sg
from paper_1511_06416_b200.engine import Engine, StepGraphs
from paper_1511_06416_b200.io import bundled_network_path, load_network_file, pack_nibbles

net, truth = load_network_file(bundled_network_path("koller"))
cases, m = 1_000_000, 10
obs = sg.forward_sample_device(net, truth, cases, seed=1, hide_fraction=0.5, mask_seed=2)
mb = next(iter(sg.DeviceSource(obs, cases, cases)))


def warm_pcie(host):
    """Bring the PCIe link out of its low-power state (bench.py does the same)."""
    import time
    scratch = torch.empty_like(host, device="cuda")
    t = time.perf_counter()
    while time.perf_counter() - t < 0.3:
        for _ in range(8):
            scratch.copy_(host, non_blocking=True)
        torch.cuda.synchronize()


def timed(g, steps=50, host=None):
    if host is not None:
        warm_pcie(host)
    for _ in range(3):
        g.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        g.step()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps * 1e3


from paper_1511_06416_b200.io import pack_bits

for rep in range(2):
    cfg = sg.SamplerConfig(same_m=m, minibatch_size=cases, num_passes=1, seed=300, rng="joint")
    eng = Engine(net, cfg)
    for w in range(3):
        eng.visit(mb, w, m)
    shape, dt = StepGraphs.obs_geometry(5, cases, 2)
    host = torch.empty(shape, dtype=dt, pin_memory=True)
    host.copy_(pack_bits(obs[:, :cases], shape[1] * 4, 2).cpu())
    cpt_host = torch.empty(eng.pack.cells, dtype=torch.float64, pin_memory=True)
    base = 3
    for label, kw in [("plain", {}), ("readback", {"readback": [(eng.cpt, cpt_host)]}),
                      ("host_block", {"host_block": host}),
                      ("host_block+readback", {"host_block": host, "readback": [(eng.cpt, cpt_host)]})]:
        g = StepGraphs(eng, mb, m, range(base, base + 60), obs_bits=2, **kw)
        print(f"rep {rep} {label:22s} {timed(g, host=host):7.1f} us/step", flush=True)
        g.finish()
        base += 70

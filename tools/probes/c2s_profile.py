"""Dev probe: host-side profile of run() streaming C2 minibatches (c2s)."""
import cProfile
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1511_06416_b200 as sg
from paper_1511_06416_b200.io import bundled_network_path, load_network_file

net, truth = load_network_file(bundled_network_path("koller"))
B, cases = 1_000_000, 20_000_000
src = sg.HostSource.from_device_blocks(
    lambda lo, hi: sg.forward_sample_device(net, truth, hi - lo, seed=100, hide_fraction=0.5, mask_seed=200,
                                            case_base=lo)[:, :hi - lo], net.num_vars, cases, B, bits=2)
cfg = sg.SamplerConfig(same_m=10, minibatch_size=B, num_passes=3, seed=300, rng="joint",
                       accumulator_mode="exponential", exp_decay=0.9)
sg.run(net, src, cfg)  # warm
pr = cProfile.Profile()
pr.enable()
_, trace = sg.run(net, src, cfg)
pr.disable()
print([round((r.seconds - (trace.records[i - 1].seconds if i else 0)) / (cases / B) * 1e6, 1) for i, r in enumerate(trace.records)], "us/step per pass")
pstats.Stats(pr).sort_stats("tottime").print_stats(25)

import sys, numpy as np
sys.path.insert(0, '.')
import paper_1511_06416_b200 as sg
from paper_1511_06416_b200.io import bundled_network_path, load_network_file
net, truth = load_network_file(bundled_network_path("koller"))
for rng in ("numpy", "fast"):
    errs, kls = [], []
    for seed in range(8):
        obs = sg.forward_sample_device(net, truth, 50_000, seed=100 + seed, hide_fraction=0.5, mask_seed=200 + seed)
        cfg = sg.SamplerConfig(same_m=1, minibatch_size=12_500, num_passes=200, seed=300 + seed, rng=rng)
        cpts, trace = sg.run(net, sg.DeviceSource(obs, 50_000, 12_500), cfg, truth=truth)
        errs.append(sg.avg_abs_error(truth, cpts)); kls.append(sg.kl_avg(truth, cpts))
    print(rng, "err", np.round(errs, 4), "median", np.median(errs), "kl", np.round(kls, 5), "median", np.median(kls))

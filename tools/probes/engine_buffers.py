import paper_1511_06416_b200 as sg
from paper_1511_06416_b200.engine import Engine
from paper_1511_06416_b200.io import bundled_network_path, load_network_file
net, truth = load_network_file(bundled_network_path("koller"))
obs = sg.forward_sample_device(net, truth, 100000, seed=1, hide_fraction=0.5, mask_seed=2)
eng = Engine(net, sg.SamplerConfig(same_m=10, minibatch_size=100000, seed=3, rng="joint"))
for k, v in vars(eng).items():
    if hasattr(v, "numel") and hasattr(v, "element_size"):
        print(k, v.numel() * v.element_size(), tuple(v.shape))

import sys; sys.path.insert(0, '/root/repo')
import torch, numpy as np
import paper_1511_06416_b200 as sg
from paper_1511_06416_b200 import netgen
from paper_1511_06416_b200.engine import Engine
net = netgen.random_dag_network(1000, 4, 2, 4, seed=4)
truth = netgen.dirichlet_cpts(net, 1.0, seed=5)
obs = sg.forward_sample_device(net, truth, 3000, seed=104, hide_fraction=0.3, mask_seed=204)
cfg = sg.SamplerConfig(same_m=1, minibatch_size=3000, num_passes=1, seed=3, rng="fast")
eng = Engine(net, cfg)
mb = next(iter(sg.DeviceSource(obs, 3000, 3000)))
eng.visit(mb, 0, 1); torch.cuda.synchronize(); print("visit ok", eng.err.read())

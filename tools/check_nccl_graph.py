"""Dev check: an Engine with the NCCL count all-reduce hook, eager and under
StepGraphs capture, on however many ranks torchrun starts (1 is enough to
exercise capture of the collective).  Prints OK on rank 0.

  torchrun --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 tools/check_nccl_graph.py
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import torch.distributed as dist

import paper_1511_06416_b200 as sg
from paper_1511_06416_b200.engine import Engine, StepGraphs
from paper_1511_06416_b200.io import bundled_network_path, load_network_file

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
net, truth = load_network_file(bundled_network_path("koller"))
cases, m = 100_000, 10
obs = sg.forward_sample_device(net, truth, cases, seed=100, hide_fraction=0.5, mask_seed=200, case_base=rank * cases)
cfg = sg.SamplerConfig(same_m=m, minibatch_size=cases, num_passes=1, seed=300, rng="fast")
mb = next(iter(sg.DeviceSource(obs, cases, cases)))
a = Engine(net, cfg, case_base=rank * cases, comm=lambda c: dist.all_reduce(c))
b = Engine(net, cfg, case_base=rank * cases, comm=lambda c: dist.all_reduce(c))
for p in range(6):
    a.visit(mb, p, m)
b.visit(mb, 0, m)
g = StepGraphs(b, mb, m, range(1, 6))
for _ in range(5):
    g.step()
g.finish()
torch.cuda.synchronize()
ok = np.array_equal(a.cpt.cpu().numpy(), b.cpt.cpu().numpy())
# every rank holds the same CPTs (identical update from the all-reduced counts)
t = b.cpt.clone()
dist.broadcast(t, 0)
same = bool(torch.equal(t, b.cpt))
tot = a.prev_counts[0].sum().item()
# run(): the capturable NCCL hook (parallel.count_allreduce) lets Engine.run replay its
# steady-state visits as graphs with the all-reduce inside; equal to eager visits
from paper_1511_06416_b200 import parallel  # noqa: E402

comm = parallel.count_allreduce()
cfg2 = sg.SamplerConfig(same_m=m, minibatch_size=cases // 2, num_passes=4, seed=301, rng="joint")
res = []
for graphs in (False, True):
    eng = Engine(net, cfg2, case_base=rank * cases, comm=comm)
    eng.graph_replay = graphs
    cp, _ = eng.run(sg.DeviceSource(obs, cases, cases // 2))
    res.append(cp)
    if graphs:
        used = eng.graphs_ok()
run_ok = all(np.array_equal(x, y) for x, y in zip(res[0].tables, res[1].tables))
if rank == 0:
    print("OK" if ok and same and run_ok and used else "MISMATCH", "graph==eager", ok, "ranks agree", same,
          "run graphs==eager", run_ok, "graphs used", used, "count mass", tot, "expected",
          net.num_vars * m * cases * world, flush=True)
dist.destroy_process_group()

"""Row (e) end to end on the device: two ranks, each sweeping its case shard
on cuda:0 and all-reducing the count tables (gloo over CUDA tensors -- a host
collective, so no kernel waits on another rank's kernel), reproduce the
single-rank run over the whole minibatch bit for bit (FAST counters use
global case ids; every rank applies the same Dirichlet draw)."""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

sg = pytest.importorskip("paper_1511_06416_b200")


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(kind):
    from paper_1511_06416_b200 import netgen
    from paper_1511_06416_b200.io import bundled_network_path, load_network_file

    if kind == "koller":  # packed-lane path
        net, truth = load_network_file(bundled_network_path("koller"))
        return net, truth, 6_000, 10
    net = netgen.random_dag_network(200, max_parents=4, seed=21)  # generic large-network path
    return net, netgen.dirichlet_cpts(net, 1.0, seed=22), 3_000, 3


def _run(kind, rng, lo, hi, comm, exchange=None, passes=3):
    from paper_1511_06416_b200.engine import Engine

    net, truth, cases, m = _problem(kind)
    obs = sg.forward_sample_device(net, truth, hi - lo, seed=40, hide_fraction=0.4, mask_seed=41, case_base=lo)
    cfg = sg.SamplerConfig(same_m=m, minibatch_size=hi - lo, num_passes=passes, seed=42, rng=rng)
    eng = Engine(net, cfg, case_base=lo, comm=comm, exchange=exchange)
    mb = next(iter(sg.DeviceSource(obs, hi - lo, hi - lo)))
    for p in range(passes):
        eng.visit(mb, p, m)
    torch.cuda.synchronize()
    assert eng.err.read() == 0
    return eng.cpt.cpu().numpy(), eng.prev_counts[0].cpu().numpy()


def _worker(rank, world, port, kind, rng, out):
    import torch.distributed as dist

    from paper_1511_06416_b200.parallel import count_allreduce, rank_prefix_exchange, shard_range

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    _, _, cases, _ = _problem(kind)
    lo, hi = shard_range(cases, world, rank)
    out[rank] = _run(kind, rng, lo, hi, count_allreduce(), rank_prefix_exchange())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("kind,rng", [("koller", "fast"), ("koller", "joint"), ("dag200", "fast"), ("koller", "numpy"),
                                      ("dag200", "numpy")])
def test_two_ranks_equal_one_rank(kind, rng):
    """NUMPY mode needs the global rank prefixes (parallel.rank_prefix_exchange):
    with them the sharded run is bit-identical to the reference's own draws."""
    import torch.multiprocessing as mp

    _, _, cases, _ = _problem(kind)
    manager = mp.get_context("spawn").Manager()
    out = manager.dict()
    mp.start_processes(_worker, args=(2, _free_port(), kind, rng, out), nprocs=2, join=True, start_method="spawn")
    cpt1, counts1 = _run(kind, rng, 0, cases, None)
    for r in (0, 1):
        cpt, counts = out[r]
        np.testing.assert_array_equal(counts, counts1)
        np.testing.assert_array_equal(cpt, cpt1)

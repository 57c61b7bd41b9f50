"""Multi-rank host logic on CPU (gloo, world size 2): case sharding plus the
count all-reduce reproduce the single-rank tally of the global minibatch, and
the shard-local FAST counters use global case ids."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, dense, values_after, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1511_06416_b200.parallel import count_allreduce, shard_range

    net, _ = O.koller()
    lo, hi = shard_range(dense.shape[1], world, rank)
    # this rank's lanes after the sweep (m = 2 replicas of its cases)
    m = 2
    B = dense.shape[1]
    lanes = np.concatenate([values_after[:, r * B + lo: r * B + hi] for r in range(m)], axis=1)
    tab = O.tally(net, lanes, np.ones(lanes.shape[1]))
    flat = torch.from_numpy(np.concatenate([t.ravel() for t in tab]).astype(np.int64))
    count_allreduce()(flat)
    out[rank] = flat.numpy().copy()
    dist.barrier()
    dist.destroy_process_group()


def test_shard_range_partitions_cases():
    from paper_1511_06416_b200.parallel import shard_range

    for n in (1, 7, 100, 1001):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


def test_two_rank_count_allreduce_equals_single_rank_tally():
    net, truth = O.koller()
    dense = O.mask_dense(O.forward_sample(net, truth, 301, 5), 0.5, 6)
    values, missing = O.replicate(dense, 2)
    O.init_latent(net, values, missing, 9, 0, 0)
    O.gibbs_pass(net, O.greedy_coloring(net), truth, values, missing, 77)
    full = O.tally(net, values, np.ones(values.shape[1]))
    expect = np.concatenate([t.ravel() for t in full]).astype(np.int64)
    manager = mp.Manager()
    out = manager.dict()
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, dense, values, out), nprocs=2, join=True, start_method="fork")
    assert set(out.keys()) == {0, 1}
    np.testing.assert_array_equal(out[0], expect)
    np.testing.assert_array_equal(out[1], expect)

"""Out-of-core sources anchored to the CPU oracle.

HostSource (pinned host blocks, copy stream one minibatch ahead) and
BinaryFileSource (.sgb file -> pinned buffer -> device, 4-/2-bit rows
decoded on the device) are the reference's minibatch-source protocol
(sampler.py:393-398, FileSource io.py:156-240).  With the numpy stream and
MAP updates a run is a deterministic function of the data, so a streamed run
must reproduce the oracle's run (oracle.run, the restatement of
sampler.py:385-495 pinned to reference fixtures) bit for bit: final CPTs and
every pass's kl_avg, in moving-sum and exponential modes, with a padded final
block and SAME replication.
"""

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu

sg = pytest.importorskip("paper_1511_06416_b200")

CASES = [
    dict(accumulator_mode="moving_sum", same_m=3, num_passes=3),
    dict(accumulator_mode="exponential", exp_decay=0.7, same_m=2, num_passes=3),
    dict(accumulator_mode="moving_sum", same_m=[(1, 1), (2, 2)], num_passes=3, sweeps_per_minibatch=2),
]


def _data(koller, cases=2_500):
    net, truth = koller
    obs = sg.forward_sample_device(net, truth, cases, seed=140, hide_fraction=0.5, mask_seed=240)
    return obs[:, :cases].cpu().numpy().astype(np.int32)


def _oracle(dense, mb, kw):
    onet, otruth = O.koller()
    args = dict(kw)
    return O.run(onet, dense, minibatch_size=mb, map_estimate=True, seed=21, truth=otruth, **args)


def _check(cpts, trace, ref):
    for a, b in zip(cpts.tables, ref.cpts):
        np.testing.assert_array_equal(a, b)
    assert [r.kl_avg for r in trace.records] == ref.kl


@pytest.mark.parametrize("kw", CASES, ids=["moving", "exponential", "anneal_sweeps2"])
def test_host_source_equals_oracle(koller, kw):
    net, truth = koller
    dense = _data(koller)
    mb = 1_024  # two full blocks and a padded third
    cfg = sg.SamplerConfig(minibatch_size=mb, map_estimate=True, seed=21, **kw)
    cpts, trace = sg.run(net, sg.HostSource.from_dense(dense, mb), cfg, truth=truth)
    _check(cpts, trace, _oracle(dense, mb, kw))


@pytest.mark.parametrize("encoding", ["int8", "nibble", "crumb"])
@pytest.mark.parametrize("kw", CASES[:2], ids=["moving", "exponential"])
def test_binary_file_source_equals_oracle(tmp_path, koller, encoding, kw):
    from paper_1511_06416_b200 import io

    net, truth = koller
    dense = _data(koller)
    mb = 1_024
    path = tmp_path / f"obs_{encoding}.sgb"
    io.write_binary(path, dense, mb, encoding)
    cfg = sg.SamplerConfig(minibatch_size=mb, map_estimate=True, seed=21, **kw)
    cpts, trace = sg.run(net, io.BinaryFileSource(path), cfg, truth=truth)
    _check(cpts, trace, _oracle(dense, mb, kw))


def test_large_network_streamed_equals_oracle():
    """The generic (large-network) kernels behind a streamed source: a 120-node
    random DAG, cards 2-4, numpy stream, MAP, exponential accumulator."""
    from paper_1511_06416_b200 import io, netgen

    net = netgen.random_dag_network(120, max_parents=4, min_card=2, max_card=4, seed=11)
    truth = netgen.dirichlet_cpts(net, 1.0, seed=12)
    obs = sg.forward_sample_device(net, truth, 700, seed=13, hide_fraction=0.3, mask_seed=14)
    dense = obs[:, :700].cpu().numpy().astype(np.int32)
    onet = O.make_net(list(net.cardinalities), [(p, c) for c in range(net.num_vars) for p in net.parents[c]])
    kw = dict(accumulator_mode="exponential", exp_decay=0.8, same_m=2, num_passes=2)
    ref = O.run(onet, dense, minibatch_size=256, map_estimate=True, seed=15, truth=truth.tables, **kw)
    cfg = sg.SamplerConfig(minibatch_size=256, map_estimate=True, seed=15, **kw)
    cpts, trace = sg.run(net, sg.HostSource.from_dense(dense, 256), cfg, truth=truth)
    _check(cpts, trace, ref)
    path = None
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        path = f"{td}/dag.sgb"
        io.write_binary(path, dense, 256, "nibble")
        cpts, trace = sg.run(net, io.BinaryFileSource(path), cfg, truth=truth)
        _check(cpts, trace, ref)

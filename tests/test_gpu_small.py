"""The packed-lane path (sg_small.cu) against the generic sweep (sg_sweep.cu).

Both implement the FAST RNG mode with the same Philox4x32 counters and the
same conditional tables, so for the same inputs they must agree bit for bit:
lane states after every visit, count tables, and the CPT trajectory.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

sg = pytest.importorskip("paper_1511_06416_b200")


def _engines(net, cfg):
    from paper_1511_06416_b200.engine import Engine

    a = Engine(net, cfg, small=True)
    b = Engine(net, cfg, small=False)
    assert a.use_small and not b.use_small
    return a, b


def _compare(net, obs, cases, mb_size, m, visits=2, seed=5, map_estimate=False):
    cfg = sg.SamplerConfig(same_m=m, minibatch_size=mb_size, num_passes=1, seed=seed, rng="fast",
                           map_estimate=map_estimate)
    a, b = _engines(net, cfg)
    src = sg.DeviceSource(obs, cases, mb_size)
    for p in range(visits):
        for mb in src:
            a.visit(mb, p, m)
            b.visit(mb, p, m)
            torch.cuda.synchronize()
            ca = a.prev_counts[mb.index].cpu().numpy()
            cb = b.prev_counts[mb.index].cpu().numpy()
            np.testing.assert_array_equal(ca, cb)
            sa = a.lane_states(mb.index)[:, :, :mb.size].cpu().numpy()
            sb = b.lane_states(mb.index)[:, :, :mb.size].cpu().numpy()
            np.testing.assert_array_equal(sa, sb)
        np.testing.assert_array_equal(a.cpt.cpu().numpy(), b.cpt.cpu().numpy())
    assert a.err.read() == 0 and b.err.read() == 0


@pytest.mark.parametrize("m", [1, 3, 4, 10])
def test_koller_packed_equals_generic(koller, m):
    net, truth = koller
    cases = 20_000
    obs = sg.forward_sample_device(net, truth, cases, seed=11, hide_fraction=0.5, mask_seed=12)
    _compare(net, obs, cases, cases, m)


def test_koller_padding_and_several_minibatches(koller):
    net, truth = koller
    cases = 5_000
    obs = sg.forward_sample_device(net, truth, cases, seed=1, hide_fraction=0.4, mask_seed=2)
    _compare(net, obs, cases, 1_536, 5, visits=3, map_estimate=True)


@pytest.mark.parametrize("small", [True, False])
def test_graph_replay_equals_eager_visits(koller, small):
    """StepGraphs replays the same kernels with the same keys as Engine.visit."""
    from paper_1511_06416_b200.engine import Engine, StepGraphs

    net, truth = koller
    cases, m = 20_000, 10
    obs = sg.forward_sample_device(net, truth, cases, seed=21, hide_fraction=0.5, mask_seed=22)
    cfg = sg.SamplerConfig(same_m=m, minibatch_size=cases, num_passes=1, seed=9, rng="fast")
    mb = next(iter(sg.DeviceSource(obs, cases, cases)))
    a = Engine(net, cfg, small=small)
    b = Engine(net, cfg, small=small)
    for p in range(6):
        a.visit(mb, p, m)
    b.visit(mb, 0, m)
    g = StepGraphs(b, mb, m, range(1, 6), obs_buffer=obs)
    for _ in range(5):
        g.step()
    g.finish()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(a.cpt.cpu().numpy(), b.cpt.cpu().numpy())
    np.testing.assert_array_equal(a.total.cpu().numpy(), b.total.cpu().numpy())
    np.testing.assert_array_equal(a.prev_counts[0].cpu().numpy(), b.prev_counts[0].cpu().numpy())
    np.testing.assert_array_equal(a.lane_states(0)[:, :, :cases].cpu().numpy(),
                                  b.lane_states(0)[:, :, :cases].cpu().numpy())


@pytest.mark.parametrize("map_estimate", [False, True])
def test_packed_only_tables_equal_two_stage_build(koller, map_estimate):
    """The step tail's packed words built straight from the CPTs
    (SG_FINISH_PACKED_ONLY) equal sg_build_tables -> sg_small_tables."""
    from paper_1511_06416_b200 import _lib
    from paper_1511_06416_b200.device import stream_handle

    net, truth = koller
    cases, m = 10_000, 6
    obs = sg.forward_sample_device(net, truth, cases, seed=41, hide_fraction=0.5, mask_seed=42)
    cfg = sg.SamplerConfig(same_m=m, minibatch_size=cases, num_passes=1, seed=23, rng="fast",
                           map_estimate=map_estimate)
    a, _ = _engines(net, cfg)
    mb = next(iter(sg.DeviceSource(obs, cases, cases)))
    for p in range(3):
        a.visit(mb, p, m)
        ptab = torch.empty_like(a.ptab)
        ftab = torch.empty_like(a.ftab)
        stab = torch.zeros_like(a.stab)
        s = stream_handle()
        _lib.call("sg_build_tables", a.pack.ref, a.cpt.data_ptr(), ptab.data_ptr(), ftab.data_ptr(), s)
        _lib.call("sg_small_tables", a.pack.ref, a.pack.small_ref, ftab.data_ptr(), stab.data_ptr(), s)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(a.stab.cpu().numpy(), stab.cpu().numpy())
        assert int(a.ftab[-1]) == int(ftab[-1])


def test_graph_host_uploads_equal_eager_visits(koller):
    """Graph replays fed host minibatches (double-buffered copy-stream uploads)
    match eager visits bit for bit."""
    from paper_1511_06416_b200.engine import Engine, StepGraphs

    net, truth = koller
    cases, m = 30_000, 4
    obs = sg.forward_sample_device(net, truth, cases, seed=31, hide_fraction=0.5, mask_seed=32)
    cfg = sg.SamplerConfig(same_m=m, minibatch_size=cases, num_passes=1, seed=17, rng="fast")
    mb = next(iter(sg.DeviceSource(obs, cases, cases)))
    host = torch.empty((net.num_vars, cases), dtype=torch.int8, pin_memory=True)
    host.copy_(obs[:, :cases])
    hmb = sg.Minibatch(index=0, values=host, weights=np.ones(cases), num_real=cases)
    a = Engine(net, cfg)
    b = Engine(net, cfg)
    for p in range(7):
        a.visit(mb, p, m)
    b.visit(mb, 0, m)
    g = StepGraphs(b, mb, m, range(1, 7))
    for _ in range(6):
        g.step(hmb)
    g.finish()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(a.cpt.cpu().numpy(), b.cpt.cpu().numpy())
    np.testing.assert_array_equal(a.prev_counts[0].cpu().numpy(), b.prev_counts[0].cpu().numpy())
    np.testing.assert_array_equal(a.lane_states(0)[:, :, :cases].cpu().numpy(),
                                  b.lane_states(0)[:, :, :cases].cpu().numpy())
    assert b.err.read() == 0


def test_random_small_networks_packed_equals_generic():
    rng = np.random.default_rng(77)
    done = 0
    while done < 6:
        n = int(rng.integers(2, 6))
        cards = [int(rng.integers(2, 5)) for _ in range(n)]
        order = rng.permutation(n)
        edges = [(int(order[i]), int(order[j])) for i in range(n) for j in range(i + 1, n) if rng.random() < 0.5]
        net = sg.build_network(cards, edges)
        from paper_1511_06416_b200.device import netpack

        if netpack(net).small is None:
            continue
        truth = sg.CptSet([rng.dirichlet(np.ones(net.cardinalities[v]), size=net.table_shape(v)[0])
                           for v in range(n)])
        cases = 3_000
        obs = sg.forward_sample_device(net, truth, cases, seed=int(rng.integers(1 << 30)), hide_fraction=0.5,
                                       mask_seed=int(rng.integers(1 << 30)))
        _compare(net, obs, cases, cases, int(rng.integers(1, 9)))
        done += 1

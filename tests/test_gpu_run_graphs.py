"""run() replays steady-state visits as CUDA graphs (Engine.run); the results
are bit-identical to eager visits in every RNG mode, accumulator schedule and
source kind, and the numpy-mode graphs stay bit-exact with the oracle."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

sg = pytest.importorskip("paper_1511_06416_b200")


def _run(net, source, cfg, truth, graphs):
    engines = []

    def hook(e):
        e.graph_replay = graphs
        engines.append(e)

    cpts, trace = sg.run(net, source, cfg, truth=truth, engine_hook=hook)
    return cpts, trace, engines[0]


CASES = [
    dict(rng="numpy", same_m=3, map_estimate=True),
    dict(rng="numpy", same_m=[(1, 2), (3, 3)], sweeps_per_minibatch=2),
    dict(rng="fast", same_m=4),
    dict(rng="fast", same_m=2, map_estimate=True, sweeps_per_minibatch=2),
    dict(rng="joint", same_m=10),
    dict(rng="joint", same_m=[(2, 2), (5, 4)]),
]


@pytest.mark.parametrize("kw", CASES, ids=[str(i) for i in range(len(CASES))])
def test_graph_replay_equals_eager_koller(koller, kw):
    net, truth = koller
    cases = 5000  # minibatch 1024: four full blocks + a padded fifth
    obs = sg.forward_sample_device(net, truth, cases, seed=5, hide_fraction=0.5, mask_seed=6)
    cfg = sg.SamplerConfig(minibatch_size=1024, num_passes=6, seed=9, **kw)
    a, ta, ea = _run(net, sg.DeviceSource(obs, cases, 1024), cfg, truth, False)
    b, tb, eb = _run(net, sg.DeviceSource(obs, cases, 1024), cfg, truth, True)
    for x, y in zip(a.tables, b.tables):
        np.testing.assert_array_equal(x, y)
    assert [r.kl_avg for r in ta.records] == [r.kl_avg for r in tb.records]
    assert [r.vars_sampled for r in ta.records] == [r.vars_sampled for r in tb.records]
    assert ta.memory.latent_bytes == tb.memory.latent_bytes
    assert ta.memory.accumulator_bytes == tb.memory.accumulator_bytes


def test_graph_replay_numpy_map_matches_oracle(koller):
    """The replayed numpy-stream sweeps (device-hashed keys) reproduce the CPU oracle."""
    import oracle as O

    net, truth = koller
    cases = 3000
    obs = sg.forward_sample_device(net, truth, cases, seed=11, hide_fraction=0.5, mask_seed=12)
    cfg = sg.SamplerConfig(same_m=2, minibatch_size=1000, num_passes=4, map_estimate=True, seed=13)
    cpts, trace, eng = _run(net, sg.DeviceSource(obs, cases, 1000), cfg, truth, True)
    onet, otruth = O.koller()
    ref = O.run(onet, obs[:, :cases].cpu().numpy().astype(np.int32), same_m=2, minibatch_size=1000, num_passes=4,
                map_estimate=True, seed=13, truth=otruth)
    for x, y in zip(cpts.tables, ref.cpts):
        np.testing.assert_array_equal(x, y)
    assert [r.kl_avg for r in trace.records] == ref.kl


def test_graph_replay_large_network_and_host_blocks():
    """Generic path (200-variable DAG), numpy and fast streams, minibatches fed from
    host int32 blocks (DataMatrix) -- the graphs refill private buffers each visit."""
    from paper_1511_06416_b200 import netgen

    net = netgen.random_dag_network(200, max_parents=4, seed=21)
    truth = netgen.dirichlet_cpts(net, 1.0, seed=22)
    obs = sg.forward_sample_device(net, truth, 1500, seed=3, hide_fraction=0.3, mask_seed=4)
    dm = sg.DataMatrix.from_dense(obs[:, :1500].cpu().numpy().astype(np.int32))
    for rng in ("numpy", "fast"):
        cfg = sg.SamplerConfig(same_m=2, minibatch_size=512, num_passes=3, seed=7, rng=rng)
        a, ta, _ = _run(net, dm, cfg, truth, False)
        b, tb, _ = _run(net, dm, cfg, truth, True)
        for x, y in zip(a.tables, b.tables):
            np.testing.assert_array_equal(x, y)
        assert [r.kl_avg for r in ta.records] == [r.kl_avg for r in tb.records]


def test_trace_times_are_device_events(koller):
    net, truth = koller
    obs = sg.forward_sample_device(net, truth, 4096, seed=1, hide_fraction=0.5, mask_seed=2)
    cfg = sg.SamplerConfig(same_m=5, minibatch_size=4096, num_passes=5, seed=1, rng="joint")
    _, trace, eng = _run(net, sg.DeviceSource(obs, 4096, 4096), cfg, None, True)
    secs = [r.seconds for r in trace.records]
    assert all(b >= a for a, b in zip(secs, secs[1:])) and secs[0] > 0
    assert all(r.vars_per_sec and r.vars_per_sec > 0 for r in trace.records)
    assert sg.throughput(trace).overall > 0


@pytest.mark.parametrize("rng,src", [("joint", "device"), ("joint", "host"), ("fast", "device"), ("joint", "sgb")])
def test_stream_graphs_equal_eager(koller, tmp_path, rng, src):
    """Exponential accumulator on the packed / joint path: fresh visits replayed as
    stream graphs (prepare + sweep + tail per replay, the block copied into the
    graph each visit) equal eager visits bit for bit -- device, pinned-host and
    .sgb (2-bit, disk) sources, with a padded last block run eagerly."""
    from paper_1511_06416_b200 import io

    net, truth = koller
    cases = 5000
    obs = sg.forward_sample_device(net, truth, cases, seed=15, hide_fraction=0.5, mask_seed=16)
    cfg = sg.SamplerConfig(same_m=10, minibatch_size=1024, num_passes=4, seed=19, rng=rng,
                           accumulator_mode="exponential", exp_decay=0.9)

    def source():
        if src == "device":
            return sg.DeviceSource(obs, cases, 1024)
        if src == "host":
            return sg.HostSource.from_dense(obs[:, :cases].cpu(), 1024)
        path = tmp_path / "c.sgb"
        if not path.exists():
            io.write_binary(path, obs[:, :cases].cpu().numpy().astype(np.int32), 1024, "crumb")
        return io.BinaryFileSource(path)

    a, ta, _ = _run(net, source(), cfg, truth, False)
    b, tb, _ = _run(net, source(), cfg, truth, True)
    for x, y in zip(a.tables, b.tables):
        np.testing.assert_array_equal(x, y)
    assert [r.kl_avg for r in ta.records] == [r.kl_avg for r in tb.records]


def test_stream_graphs_sample_the_streamed_blocks(koller):
    """Every replay samples the block it was given: two different data sets through
    the same stream graphs give the runs of those data sets."""
    from paper_1511_06416_b200.engine import Engine, StreamGraphs

    net, truth = koller
    cfg = sg.SamplerConfig(same_m=4, minibatch_size=2048, num_passes=1, seed=3, rng="joint",
                           accumulator_mode="exponential", exp_decay=0.5)
    d1 = sg.forward_sample_device(net, truth, 2048, seed=1, hide_fraction=0.4, mask_seed=2)
    d2 = sg.forward_sample_device(net, truth, 2048, seed=7, hide_fraction=0.4, mask_seed=8)
    mbs = [next(iter(sg.DeviceSource(d, 2048, 2048))) for d in (d1, d2, d1)]
    eager = Engine(net, cfg)
    for k, mb in enumerate(mbs):
        eager.visit(mb, k, 4)
    graphed = Engine(net, cfg)
    graphed.visit(mbs[0], 0, 4)
    g = StreamGraphs(graphed, 2048, 4, [(1, 0), (2, 0)])
    g.step(mbs[1])
    g.step(mbs[2])
    torch.cuda.synchronize()
    assert torch.equal(eager.cpt, graphed.cpt) and torch.equal(eager.total, graphed.total)


@pytest.mark.parametrize("n", [60, 400])
def test_cpt_readback_stored_by_the_tail(n):
    """StepGraphs(readback=[(cpt, pinned)]): the step tail stores the new CPTs
    in the pinned tensor itself (sg_finish.cpt_host) -- the one-CTA tail and
    the multi-launch tail of a model above its cell limit alike."""
    from paper_1511_06416_b200 import netgen
    from paper_1511_06416_b200.engine import Engine, StepGraphs

    net = netgen.random_dag_network(n, max_parents=4, seed=31)
    truth = netgen.dirichlet_cpts(net, 1.0, seed=32)
    cases = 2048
    obs = sg.forward_sample_device(net, truth, cases, seed=5, hide_fraction=0.3, mask_seed=6)
    cfg = sg.SamplerConfig(same_m=2, minibatch_size=cases, num_passes=1, seed=9, rng="fast")
    mb = next(iter(sg.DeviceSource(obs, cases, cases)))
    eng = Engine(net, cfg)
    eng.visit(mb, 0, 2)
    host = torch.zeros(eng.pack.cells, dtype=torch.float64, pin_memory=True)
    g = StepGraphs(eng, mb, 2, range(1, 4), readback=[(eng.cpt, host)])
    for _ in range(3):
        g.step()
        torch.cuda.synchronize()
        np.testing.assert_array_equal(host.numpy(), eng.cpt.cpu().numpy())
    g.finish()
    assert (eng.pack.cells > 4096) == (n == 400)

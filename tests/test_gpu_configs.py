"""Parity at the network shapes of BASELINE configs C3 (MOOC-shaped) and C4
(random DAG, 1000 nodes, in-degree <= 4, cards 2-4, 30 % missing).

* numpy-RNG mode, bit-exact against the oracle (which tests/golden pins to the
  reference, including the 120-node DAG and MOOC fixtures): one sweep of the
  full-size networks on a case slice, and a MAP run over several minibatches
  and passes on the 1000-node DAG -- the generic kernel, the direct
  (untabulated) draw for large blankets and the multi-launch step tail of
  models above the single-CTA size.
* FAST mode at larger case counts: size-independent properties (tally mass,
  observed cells untouched, CPT rows normalised).
"""

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu

sg = pytest.importorskip("paper_1511_06416_b200")
from paper_1511_06416_b200 import netgen  # noqa: E402


def _oracle_net(net):
    return O.make_net(list(net.cardinalities), [(p, c) for c in range(net.num_vars) for p in net.parents[c]])


@pytest.fixture(scope="module")
def c4():
    net = netgen.random_dag_network(1000, max_parents=4, min_card=2, max_card=4, seed=4)
    truth = netgen.dirichlet_cpts(net, 1.0, seed=5)
    return net, truth


@pytest.fixture(scope="module")
def c3():
    net = netgen.mooc_network(15, 319, seed=3)
    truth = netgen.dirichlet_cpts(net, 1.0, seed=6)
    return net, truth


def _sweep_vs_oracle(net, cpts, dense, m, init_seed, sweep_seed):
    onet = _oracle_net(net)
    values, missing = O.replicate(dense, m)
    O.init_latent(onet, values, missing, init_seed, 0, 0)
    batch = sg.ReplicatedBatch(m=m, base_size=dense.shape[1], values=values.copy(),
                               lane_weights=np.ones(values.shape[1]), missing_lanes=[x.copy() for x in missing])
    counts = sg.sweep(net, sg.color_graph(sg.moralize(net)), cpts, batch, sweep_seed)
    want = O.sweep(onet, O.greedy_coloring(onet), cpts.tables, values, missing, np.ones(values.shape[1]), sweep_seed)
    np.testing.assert_array_equal(batch.values, values)
    for a, b in zip(counts.tables, want):
        np.testing.assert_array_equal(a, b)


def test_c4_colouring_matches_oracle(c4):
    net, _ = c4
    groups = sg.color_graph(sg.moralize(net)).groups
    assert [list(g) for g in groups] == O.greedy_coloring(_oracle_net(net))


def test_c4_sweep_bit_exact(c4):
    net, truth = c4
    obs = sg.forward_sample_device(net, truth, 1500, seed=104, hide_fraction=0.3, mask_seed=204)
    dense = obs[:, :1500].cpu().numpy().astype(np.int32)
    _sweep_vs_oracle(net, truth, dense, 1, 304, 9001)


def test_c4_replica_groups_bit_exact(c4):
    """n x m too large for one tile of all replicas (1000 x 10): the sweep
    splits the replicas into groups (grid y) -- still bit-exact."""
    net, truth = c4
    obs = sg.forward_sample_device(net, truth, 700, seed=106, hide_fraction=0.3, mask_seed=206)
    dense = obs[:, :700].cpu().numpy().astype(np.int32)
    _sweep_vs_oracle(net, truth, dense, 10, 305, 9003)


def test_c3_sweep_bit_exact(c3):
    net, truth = c3
    obs = netgen.mooc_observations(net, truth, 4000, 15, density=0.022, seed=103)
    dense = obs[:, :4000].cpu().numpy().astype(np.int32)
    assert (dense[:15] < 0).all()
    _sweep_vs_oracle(net, truth, dense, 5, 303, 9002)


def test_c4_map_run_bit_exact(c4):
    """Three minibatches (last one padded), two passes, moving sum, posterior
    mean: the 1000-node model (72k-cell class) exceeds the single-CTA tail, so
    this exercises the multi-launch step tail."""
    net, truth = c4
    cases = 1300
    obs = sg.forward_sample_device(net, truth, cases, seed=110, hide_fraction=0.3, mask_seed=210)
    dense = obs[:, :cases].cpu().numpy().astype(np.int32)
    cfg = sg.SamplerConfig(same_m=1, minibatch_size=500, num_passes=2, map_estimate=True, seed=310)
    cpts, trace = sg.run(net, sg.DataMatrix.from_dense(dense), cfg, truth=truth)
    res = O.run(_oracle_net(net), dense, same_m=1, minibatch_size=500, num_passes=2, map_estimate=True, seed=310,
                truth=truth.tables)
    for a, b in zip(cpts.tables, res.cpts):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal([r.kl_avg for r in trace.records], res.kl)


def _fast_properties(net, obs, cases, m, mb_size):
    from paper_1511_06416_b200.engine import Engine

    cfg = sg.SamplerConfig(same_m=m, minibatch_size=mb_size, num_passes=1, seed=7, rng="fast")
    eng = Engine(net, cfg)
    src = sg.DeviceSource(obs, cases, mb_size)
    for mb in src:
        eng.visit(mb, 0, m)
        torch.cuda.synchronize()
        counts = eng.prev_counts[mb.index].cpu().numpy()
        off = eng.pack.layout.cpt_off
        for v in range(net.num_vars):
            assert counts[off[v]:off[v + 1]].sum() == m * mb.num_real
        st = eng.lane_states(mb.index)[:, :, :mb.num_real]
        o = mb.values[:, :mb.num_real]
        lat = st < 0
        assert bool(((o >= 0).unsqueeze(1) == ~lat).all())
        assert bool(((st & 0x7F) == o.clamp(min=0).unsqueeze(1))[~lat].all())
    assert eng.err.read() == 0
    cpt = eng.current_cpts()
    for t in cpt.tables:
        np.testing.assert_allclose(t.sum(axis=1), 1.0, atol=1e-12)


def test_c3_fast_mode_properties(c3):
    net, truth = c3
    cases = 131_010  # 4,367 students x 30
    obs = netgen.mooc_observations(net, truth, cases, 15, density=0.022, seed=113)
    _fast_properties(net, obs, cases, 5, 65_536)


def test_c4_fast_mode_properties(c4):
    net, truth = c4
    cases = 200_000
    obs = sg.forward_sample_device(net, truth, cases, seed=114, hide_fraction=0.3, mask_seed=214)
    _fast_properties(net, obs, cases, 1, 100_000)


@pytest.mark.parametrize("acc", ["exponential", "moving_sum"])
def test_host_source_streaming_equals_device_source(c4, acc):
    """Out-of-core streaming (HostSource: pinned host blocks, copy stream one
    minibatch ahead, replayed twice) gives exactly the run of a device-resident
    source over the same (duplicated) data."""
    net, truth = c4
    cases, mb = 3_072, 1_024
    obs = sg.forward_sample_device(net, truth, cases, seed=120, hide_fraction=0.3, mask_seed=220)
    dense = obs[:, :cases].cpu()
    host = sg.HostSource.from_dense(dense, mb, cycle=2)
    # the device source sees the two replays as one matrix of twice the cases
    devsrc = sg.DeviceSource(torch.cat([dense, dense], dim=1).cuda(), 2 * cases, mb)
    cfg = sg.SamplerConfig(same_m=3, minibatch_size=mb, num_passes=2, seed=11, rng="fast",
                           accumulator_mode=acc, exp_decay=0.9)
    a, _ = sg.run(net, host, cfg)
    b, _ = sg.run(net, devsrc, cfg)
    for x, y in zip(a.tables, b.tables):
        np.testing.assert_array_equal(x, y)


def test_host_source_padding_equals_matrix_source(c4):
    """A final partial block (padded with missing cells of weight 0) streams
    exactly like the reference-style host matrix source."""
    net, truth = c4
    cases, mb = 2_500, 1_024
    obs = sg.forward_sample_device(net, truth, cases, seed=121, hide_fraction=0.3, mask_seed=221)
    dense = obs[:, :cases].cpu().numpy()
    cfg = sg.SamplerConfig(same_m=2, minibatch_size=mb, num_passes=2, seed=12, rng="fast",
                           accumulator_mode="exponential", exp_decay=0.8)
    a, _ = sg.run(net, sg.HostSource.from_dense(dense, mb), cfg)
    b, _ = sg.run(net, sg.DataMatrix.from_dense(dense.astype(np.int32)), cfg)
    for x, y in zip(a.tables, b.tables):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("encoding", ["int8", "nibble", "crumb"])
def test_binary_file_source_equals_matrix_source(tmp_path, koller, encoding):
    """An .sgb file streamed from disk (4-/2-bit rows decoded on the device)
    drives exactly the run of the in-memory data, padding included."""
    from paper_1511_06416_b200 import io

    net, truth = koller
    cases, mb = 5_000, 1_024
    dense = sg.forward_sample_device(net, truth, cases, seed=130, hide_fraction=0.4, mask_seed=230)[:, :cases]
    dense = dense.cpu().numpy().astype(np.int32)
    path = tmp_path / "obs.sgb"
    io.write_binary(path, dense, mb, encoding)
    for rng in ("numpy", "fast"):
        cfg = sg.SamplerConfig(same_m=3, minibatch_size=mb, num_passes=2, seed=13, rng=rng)
        a, _ = sg.run(net, io.BinaryFileSource(path), cfg)
        b, _ = sg.run(net, sg.DataMatrix.from_dense(dense), cfg)
        for x, y in zip(a.tables, b.tables):
            np.testing.assert_array_equal(x, y)


def test_unpack_nibbles_kernel():
    from paper_1511_06416_b200 import _lib
    from paper_1511_06416_b200.device import stream_handle

    rng = np.random.default_rng(4)
    rows, cases, ldp, ldo = 5, 1000, 512, 1024
    vals = rng.integers(-1, 15, size=(rows, 2 * ldp)).astype(np.int64)
    nib = np.where(vals < 0, 15, vals).astype(np.uint8)
    packed = torch.from_numpy((nib[:, 0::2] | (nib[:, 1::2] << 4)).astype(np.uint8)).cuda()
    out = torch.full((rows, ldo), 99, dtype=torch.int8, device="cuda")
    _lib.call("sg_unpack_nibbles", packed.data_ptr(), ldp, out.data_ptr(), ldo, rows, cases, stream_handle())
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    np.testing.assert_array_equal(got[:, :cases], vals[:, :cases])
    assert (got[:, cases:] == 99).all()


@pytest.mark.parametrize("hide,m", [(0.3, 1), (0.3, 6), (0.9, 3)])
def test_four_bit_states_bit_exact(hide, m):
    """Large networks with cards 5..8 keep 4-bit packed states: the big-tile
    sweep (sparse latent cells) and the lane sweep (dense, m >= 2) stay
    bit-exact against the oracle."""
    net = netgen.random_dag_network(60, max_parents=3, min_card=2, max_card=8, seed=31)
    assert max(net.cardinalities) > 4
    truth = netgen.dirichlet_cpts(net, 1.0, seed=32)
    obs = sg.forward_sample_device(net, truth, 900, seed=107, hide_fraction=hide, mask_seed=207)
    dense = obs[:, :900].cpu().numpy().astype(np.int32)
    _sweep_vs_oracle(net, truth, dense, m, 308, 9004)


@pytest.mark.parametrize("bits,max_card", [(4, 4), (2, 3)])
def test_generic_graph_with_packed_uploads_equals_eager(bits, max_card):
    """Generic-sweep StepGraphs fed packed host blocks (.sgb 4- / 2-bit form:
    unpacked + range-checked inside the graph) == eager visits on the int8
    block, bit for bit; an out-of-range state is still flagged
    (sampler.py:429-430)."""
    from paper_1511_06416_b200 import _lib
    from paper_1511_06416_b200.engine import Engine, StepGraphs
    from paper_1511_06416_b200.io import pack_bits

    net = netgen.random_dag_network(40, max_parents=4, min_card=2, max_card=max_card, seed=31)
    truth = netgen.dirichlet_cpts(net, 1.0, seed=32)
    cases, m = 20_001, 2
    obs = sg.forward_sample_device(net, truth, cases, seed=33, hide_fraction=0.3, mask_seed=34)
    cfg = sg.SamplerConfig(same_m=m, minibatch_size=cases, num_passes=1, seed=35, rng="fast")
    mb = next(iter(sg.DeviceSource(obs, cases, cases)))
    a, b = Engine(net, cfg), Engine(net, cfg)
    assert not b.use_small
    for p in range(5):
        a.visit(mb, p, m)
    b.visit(mb, 0, m)
    g = StepGraphs(b, mb, m, range(1, 6), obs_bits=bits)
    pitchp = g.obs_bufs[0].shape[1] * 8 // bits
    host = torch.empty(tuple(g.obs_bufs[0].shape), dtype=torch.uint8, pin_memory=True)
    host.copy_(torch.from_numpy(pack_bits(obs[:, :cases].cpu().numpy(), pitchp, bits)))
    hmb = sg.Minibatch(index=0, values=host, weights=np.ones(cases), num_real=cases)
    for _ in range(4):
        g.step(hmb)
    torch.cuda.synchronize()
    assert b.err.read() == 0
    np.testing.assert_array_equal(a.cpt.cpu().numpy(), b.cpt.cpu().numpy())
    np.testing.assert_array_equal(a.lane_states(0)[:, :, :cases].cpu().numpy(),
                                  b.lane_states(0)[:, :, :cases].cpu().numpy())
    bad = obs[:, :cases].cpu().numpy().copy()
    v2 = [v for v in range(net.num_vars) if net.cardinalities[v] == 2][0]
    bad[v2, cases - 1] = 2
    host.copy_(torch.from_numpy(pack_bits(bad, pitchp, bits)))
    g.step(hmb)
    torch.cuda.synchronize()
    assert b.err.read() & _lib.SG_ERR_STATE_RANGE


def test_engines_sharing_a_pack_sweep_on_two_streams():
    """Two engines of one network (one cached NetPack) sweeping concurrently on
    two streams: each rebuilds its own blanket factor tables (private sg_net
    copy), so both equal the same runs made one after the other."""
    from paper_1511_06416_b200 import netgen
    from paper_1511_06416_b200.engine import Engine

    net = netgen.random_dag_network(120, max_parents=4, min_card=2, max_card=4, seed=41)
    truth = netgen.dirichlet_cpts(net, 1.0, seed=42)
    cases = 20_000
    obs = sg.forward_sample_device(net, truth, cases, seed=43, hide_fraction=0.3, mask_seed=44)
    mb = next(iter(sg.DeviceSource(obs, cases, cases)))

    def engines():
        out = []
        for seed in (1, 2):
            cfg = sg.SamplerConfig(same_m=1, minibatch_size=cases, num_passes=1, seed=seed, rng="fast")
            out.append(Engine(net, cfg))
        return out

    seq = engines()
    for e in seq:
        for p in range(4):
            e.visit(mb, p, 1)
    torch.cuda.synchronize()
    par = engines()
    assert par[0].pack is par[1].pack
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    torch.cuda.synchronize()
    for p in range(4):
        for e, s in zip(par, streams):
            with torch.cuda.stream(s):
                e.visit(mb, p, 1)
    torch.cuda.synchronize()
    for a, b in zip(seq, par):
        np.testing.assert_array_equal(a.cpt.cpu().numpy(), b.cpt.cpu().numpy())
        np.testing.assert_array_equal(a.lane_states(0).cpu().numpy(), b.lane_states(0).cpu().numpy())

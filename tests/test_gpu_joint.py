"""The joint sweep (rng="joint", csrc/sg_small.cu) against its NumPy restatement.

tests/fast_stream.py restates the joint tables (the colour-ordered product of
the reference's full conditionals, sampler.py:217-284, tabulated per latent
pattern and lane word) and the draw (one FAST Philox word per lane, first
alias entry of its row, csrc joint_alias_row).  The device must match both bit for bit: the blob rows
after every CPT update, the lane states after a sweep, and the count tables
(the tally of the new states, model.py:148-165).
"""

import numpy as np
import pytest
import torch

import fast_stream as F
import oracle as O

pytestmark = pytest.mark.gpu

sg = pytest.importorskip("paper_1511_06416_b200")


def _onet(net):
    edges = [(p, c) for c in range(net.num_vars) for p in net.parents[c]]
    return O.make_net(list(net.cardinalities), edges)


def _blob_rows(eng, P):
    jp = eng.pack.joint
    blob = eng.jblob.cpu().numpy().view(np.uint32)
    head = blob[:jp.header_words]
    B = int(head[jp.patterns + P] & 0xFF)
    off = int(head[P]) // 4
    R, K = 1 << eng.pack.small.bits, 1 << B
    rows = blob[off:off + R * (K + 1)].reshape(R, K + 1)  # odd row stride: one padding word
    assert np.all(rows[:, K] == 0)
    return rows[:, :K]


def _check_tables(eng, onet, order):
    cpts = eng.pack.split(eng.cpt.cpu().numpy())
    tabs = F.joint_tables(onet, cpts, order)
    for P, (B, keep, dep, rows) in tabs.items():
        got = _blob_rows(eng, P)
        np.testing.assert_array_equal(got, rows, err_msg=f"pattern {P}")
        head = eng.jblob.cpu().numpy().view(np.uint32)
        meta = int(head[eng.pack.joint.patterns + P])
        assert meta & 0xFF == B and (meta >> 8) & 0xFF == keep


def _tally(onet, states, num_real):
    out = []
    for v in range(onet.n):
        cfg = np.zeros(states.shape[1:], dtype=np.int64)
        for p, st in zip(onet.parents[v], onet.strides(v)):
            cfg += states[p].astype(np.int64) * st
        flat = (cfg * onet.cards[v] + states[v])[:, :num_real].ravel()
        out.append(np.bincount(flat, minlength=onet.rows(v) * onet.cards[v]))
    return np.concatenate(out)


@pytest.mark.parametrize("m,map_estimate", [(1, True), (3, False), (10, False), (13, True)])
def test_koller_joint_sweep_matches_restatement(koller, m, map_estimate):
    from paper_1511_06416_b200.engine import Engine

    net, truth = koller
    onet = _onet(net)
    order = [v for g in O.greedy_coloring(onet) for v in g]
    assert order == [int(x) for x in eng_order(net)]
    cases = 6_000
    obs = sg.forward_sample_device(net, truth, cases, seed=51, hide_fraction=0.5, mask_seed=52)
    cfg = sg.SamplerConfig(same_m=m, minibatch_size=cases, num_passes=1, seed=13, rng="joint",
                           map_estimate=map_estimate)
    eng = Engine(net, cfg)
    assert eng.joint and eng.use_small
    mb = next(iter(sg.DeviceSource(obs, cases, cases)))
    latent = (obs[:, :cases] < 0).cpu().numpy()
    eng.visit(mb, 0, m)
    for p in range(1, 4):
        torch.cuda.synchronize()
        _check_tables(eng, onet, order)
        before = eng.lane_states(0)[:, :, :cases].cpu().numpy().astype(np.int64) & 0x7F
        cpts = eng.pack.split(eng.cpt.cpu().numpy())
        tabs = F.joint_tables(onet, cpts, order)
        eng.visit(mb, p, m)
        torch.cuda.synchronize()
        after = eng.lane_states(0)[:, :, :cases].cpu().numpy().astype(np.int64) & 0x7F
        key = sg.rng.derive_seed(cfg.seed, "sweep", p, 0, 0)
        want = F.joint_sweep(tabs, net.cardinalities, before, latent, key)
        np.testing.assert_array_equal(after, want)
        np.testing.assert_array_equal(eng.prev_counts[0].cpu().numpy(), _tally(onet, after, cases))
    assert eng.err.read() == 0


def eng_order(net):
    from paper_1511_06416_b200.device import netpack

    sp = netpack(net).small
    return list(sp.order)[:net.num_vars]


def test_random_small_networks_joint_tables_and_sweep():
    from paper_1511_06416_b200.device import netpack
    from paper_1511_06416_b200.engine import Engine

    rng = np.random.default_rng(91)
    done = 0
    while done < 5:
        n = int(rng.integers(2, 6))
        cards = [int(rng.integers(2, 5)) for _ in range(n)]
        order = rng.permutation(n)
        edges = [(int(order[i]), int(order[j])) for i in range(n) for j in range(i + 1, n) if rng.random() < 0.5]
        net = sg.build_network(cards, edges)
        if netpack(net).joint is None:
            continue
        truth = sg.CptSet([rng.dirichlet(np.ones(net.cardinalities[v]), size=net.table_shape(v)[0])
                           for v in range(n)])
        cases, m = 2_000, int(rng.integers(1, 9))
        obs = sg.forward_sample_device(net, truth, cases, seed=int(rng.integers(1 << 30)), hide_fraction=0.5,
                                       mask_seed=int(rng.integers(1 << 30)))
        cfg = sg.SamplerConfig(same_m=m, minibatch_size=cases, num_passes=1, seed=5, rng="joint")
        eng = Engine(net, cfg)
        onet = _onet(net)
        corder = [v for g in O.greedy_coloring(onet) for v in g]
        mb = next(iter(sg.DeviceSource(obs, cases, cases)))
        latent = (obs[:, :cases] < 0).cpu().numpy()
        eng.visit(mb, 0, m)
        torch.cuda.synchronize()
        _check_tables(eng, onet, corder)
        before = eng.lane_states(0)[:, :, :cases].cpu().numpy().astype(np.int64) & 0x7F
        tabs = F.joint_tables(onet, eng.pack.split(eng.cpt.cpu().numpy()), corder)
        eng.visit(mb, 1, m)
        torch.cuda.synchronize()
        after = eng.lane_states(0)[:, :, :cases].cpu().numpy().astype(np.int64) & 0x7F
        key = sg.rng.derive_seed(cfg.seed, "sweep", 1, 0, 0)
        np.testing.assert_array_equal(after, F.joint_sweep(tabs, net.cardinalities, before, latent, key))
        np.testing.assert_array_equal(eng.prev_counts[0].cpu().numpy(), _tally(onet, after, cases))
        done += 1


def test_joint_graph_replay_equals_eager(koller):
    from paper_1511_06416_b200.engine import Engine, StepGraphs

    net, truth = koller
    cases, m = 20_000, 10
    obs = sg.forward_sample_device(net, truth, cases, seed=21, hide_fraction=0.5, mask_seed=22)
    cfg = sg.SamplerConfig(same_m=m, minibatch_size=cases, num_passes=1, seed=9, rng="joint")
    mb = next(iter(sg.DeviceSource(obs, cases, cases)))
    a, b = Engine(net, cfg), Engine(net, cfg)
    for p in range(6):
        a.visit(mb, p, m)
    b.visit(mb, 0, m)
    g = StepGraphs(b, mb, m, range(1, 6), obs_buffer=obs)
    for _ in range(5):
        g.step()
    g.finish()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(a.cpt.cpu().numpy(), b.cpt.cpu().numpy())
    np.testing.assert_array_equal(a.prev_counts[0].cpu().numpy(), b.prev_counts[0].cpu().numpy())
    np.testing.assert_array_equal(a.lane_states(0)[:, :, :cases].cpu().numpy(),
                                  b.lane_states(0)[:, :, :cases].cpu().numpy())
    np.testing.assert_array_equal(a.jblob.cpu().numpy(), b.jblob.cpu().numpy())


def test_joint_stream_samples_the_posterior(koller):
    """Lanes with a fixed observed pattern, CPTs frozen (MAP of zero counts keeps
    them at the prior mean, so use the truth via a dedicated engine reset):
    the empirical joint distribution of the latent fields over sweeps matches
    the enumerated posterior (TV <= 0.02, test_sampler.py:141-172)."""
    from paper_1511_06416_b200.engine import Engine

    net, truth = koller
    cases, m = 4_000, 8
    obs = torch.full((net.num_vars, 4096), -1, dtype=torch.int8, device="cuda")
    obs[3] = 1  # grade observed, every other variable latent
    cfg = sg.SamplerConfig(same_m=m, minibatch_size=cases, num_passes=1, seed=3, rng="joint")
    eng = Engine(net, cfg)
    mb = next(iter(sg.DeviceSource(obs, cases, cases)))
    hist = np.zeros(2 * 2 * 2 * 2, dtype=np.int64)
    for p in range(40):
        eng.cpt.copy_(torch.from_numpy(eng.pack.flatten(truth.tables)))
        eng.tables_fresh = False
        eng.visit(mb, p, m)
        if p >= 8:
            st = eng.lane_states(0)[:, :, :cases].cpu().numpy().astype(np.int64) & 0x7F
            code = ((st[0] * 2 + st[1]) * 2 + st[2]) * 2 + st[4]
            hist += np.bincount(code.ravel(), minlength=16)
    import itertools

    exact = []
    for d, i, s, l in itertools.product(range(2), repeat=4):
        a = [d, i, s, 1, l]
        pr = 1.0
        for v in range(5):
            pr *= truth.tables[v][sg.model.parent_config_index(net, v, np.asarray(a)), a[v]]
        exact.append(pr)
    exact = np.asarray(exact) / np.sum(exact)
    tv = 0.5 * np.abs(hist / hist.sum() - exact).sum()
    assert tv <= 0.02, tv


@pytest.mark.parametrize("bits", [4, 2])
def test_joint_graph_with_4bit_uploads_equals_eager(koller, bits):
    """StepGraphs fed 4-bit host blocks (.sgb form, half the PCIe bytes) ==
    eager visits on the int8 block, bit for bit; a state >= card in the 4-bit
    block is flagged like the int8 range check (sampler.py:429-430)."""
    from paper_1511_06416_b200 import _lib
    from paper_1511_06416_b200.engine import Engine, StepGraphs
    from paper_1511_06416_b200.io import pack_bits

    net, truth = koller
    cases, m = 30_001, 10
    obs = sg.forward_sample_device(net, truth, cases, seed=61, hide_fraction=0.5, mask_seed=62)
    cfg = sg.SamplerConfig(same_m=m, minibatch_size=cases, num_passes=1, seed=17, rng="joint")
    mb = next(iter(sg.DeviceSource(obs, cases, cases)))
    a, b = Engine(net, cfg), Engine(net, cfg)
    for p in range(5):
        a.visit(mb, p, m)
    b.visit(mb, 0, m)
    g = StepGraphs(b, mb, m, range(1, 7), obs_bits=bits)
    pitch4 = g.obs_bufs[0].shape[1] * 8 // bits
    host = torch.empty(tuple(g.obs_bufs[0].shape), dtype=torch.uint8, pin_memory=True)
    host.copy_(torch.from_numpy(pack_bits(obs[:, :cases].cpu().numpy(), pitch4, bits)))
    hmb = sg.Minibatch(index=0, values=host, weights=np.ones(cases), num_real=cases)
    for _ in range(4):
        g.step(hmb)
    torch.cuda.synchronize()
    assert b.err.read() == 0
    np.testing.assert_array_equal(a.cpt.cpu().numpy(), b.cpt.cpu().numpy())
    np.testing.assert_array_equal(a.lane_states(0)[:, :, :cases].cpu().numpy(),
                                  b.lane_states(0)[:, :, :cases].cpu().numpy())
    # a bad state in the padding past the last case is not part of the minibatch
    pad = np.full((obs.shape[0], cases + 7), -1, dtype=np.int64)
    pad[:, :cases] = obs[:, :cases].cpu().numpy()
    pad[0, cases:] = 2
    host.copy_(torch.from_numpy(pack_bits(pad, pitch4, bits)))
    g.step(hmb)
    torch.cuda.synchronize()
    assert b.err.read() == 0
    bad = obs[:, :cases].cpu().numpy().copy()
    bad[0, cases - 1] = 2  # variable 0 has 2 states (2 is representable in 2 and 4 bits)
    host.copy_(torch.from_numpy(pack_bits(bad, pitch4, bits)))
    g.step(hmb)
    torch.cuda.synchronize()
    assert b.err.read() & _lib.SG_ERR_STATE_RANGE


@pytest.mark.parametrize("rng,bits,vpr,per_visit", [("joint", 4, 1, False), ("joint", 2, 1, False),
                                                    ("joint", 8, 1, False), ("fast", 8, 1, False),
                                                    ("joint", 2, 2, False), ("fast", 8, 2, False),
                                                    ("joint", 2, 2, True), ("fast", 8, 2, True)])
def test_host_fed_step_graphs_equal_eager(koller, rng, bits, vpr, per_visit):
    """StepGraphs(host_block=...): each replay uploads the next visit's pinned
    block beside the sweep and reads the CPTs back -- same results as eager
    visits, and the read-back CPTs are the engine's.  ``per_visit``: one host
    block per visit of a replay, both uploaded with one copy."""
    from paper_1511_06416_b200.engine import Engine, StepGraphs
    from paper_1511_06416_b200.io import pack_bits

    net, truth = koller
    cases, m = 20_000, 10
    obs = sg.forward_sample_device(net, truth, cases, seed=71, hide_fraction=0.5, mask_seed=72)
    cfg = sg.SamplerConfig(same_m=m, minibatch_size=cases, num_passes=1, seed=19, rng=rng)
    mb = next(iter(sg.DeviceSource(obs, cases, cases)))
    a, b = Engine(net, cfg), Engine(net, cfg)
    for p in range(5):
        a.visit(mb, p, m)
    b.visit(mb, 0, m)
    shape, dt = StepGraphs.obs_geometry(net.num_vars, cases, bits)
    host = torch.empty(shape, dtype=dt, pin_memory=True)
    if bits < 8:
        host.copy_(torch.from_numpy(pack_bits(obs[:, :cases].cpu().numpy(), shape[1] * 8 // bits, bits)))
    else:
        host.fill_(-1)
        host[:, :cases].copy_(obs[:, :cases])
    if per_visit:
        two = torch.empty((vpr, *shape), dtype=dt, pin_memory=True)
        two.copy_(host.expand(vpr, *shape))
        host = two
    cpt_host = torch.empty(b.pack.cells, dtype=torch.float64, pin_memory=True)
    g = StepGraphs(b, mb, m, range(1, 5), obs_bits=bits, host_block=host, readback=[(b.cpt, cpt_host)],
                   visits_per_replay=vpr)
    assert g.host_per_visit == per_visit
    for _ in range(4 // vpr):
        g.step()
    g.finish()
    torch.cuda.synchronize()
    assert b.err.read() == 0
    np.testing.assert_array_equal(a.cpt.cpu().numpy(), b.cpt.cpu().numpy())
    np.testing.assert_array_equal(cpt_host.numpy(), b.cpt.cpu().numpy())
    np.testing.assert_array_equal(a.prev_counts[0].cpu().numpy(), b.prev_counts[0].cpu().numpy())
    np.testing.assert_array_equal(a.lane_states(0)[:, :, :cases].cpu().numpy(),
                                  b.lane_states(0)[:, :, :cases].cpu().numpy())


def test_per_visit_host_blocks_are_each_range_checked(koller):
    """A bad state in the SECOND visit's block of a per-visit host block is
    uploaded by the merged copy into that visit's buffer and flagged."""
    from paper_1511_06416_b200 import _lib
    from paper_1511_06416_b200.engine import Engine, StepGraphs

    net, truth = koller
    cases, m = 8_192, 4
    obs = sg.forward_sample_device(net, truth, cases, seed=81, hide_fraction=0.5, mask_seed=82)
    cfg = sg.SamplerConfig(same_m=m, minibatch_size=cases, num_passes=1, seed=29, rng="joint")
    mb = next(iter(sg.DeviceSource(obs, cases, cases)))
    b = Engine(net, cfg)
    b.visit(mb, 0, m)
    shape, dt = StepGraphs.obs_geometry(net.num_vars, cases, 8)
    host = torch.full((2, *shape), -1, dtype=dt).pin_memory()
    host[:, :, :cases].copy_(obs[:, :cases].unsqueeze(0).expand(2, -1, -1))
    g = StepGraphs(b, mb, m, range(1, 13), obs_bits=8, host_block=host, visits_per_replay=2)
    for _ in range(2):
        g.step()
    torch.cuda.synchronize()
    assert b.err.read() == 0
    g.upload_done.synchronize()
    host[1, 0, 7] = 9  # variable 0 has 2 states; uploaded for visits 9 (replayed by the 5th step) and 11
    for _ in range(4):
        g.step()
    g.finish()
    torch.cuda.synchronize()
    assert b.err.read() & _lib.SG_ERR_STATE_RANGE

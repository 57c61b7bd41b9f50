"""Full-size checks at BASELINE config 2 (Koller, 1M cases, 50% hidden, m=10).

* numpy-RNG mode: one MAP pass through ``run()`` is bit-identical to the
  oracle's run at full size (init CPTs, latent init, sweep, tally, moving sum,
  posterior mean).
* fast mode: size-independent properties -- tally mass is m x cases per
  variable, observed cells never change, and the tallies agree with the
  numpy-mode tallies within sampling noise.
"""

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

sg = pytest.importorskip("paper_1511_06416_b200")

CASES = 1_000_000
M = 10


@pytest.fixture(scope="module")
def config2(koller):
    net, truth = koller
    obs = sg.forward_sample_device(net, truth, CASES, seed=100, hide_fraction=0.5, mask_seed=200)
    return net, truth, obs


def test_config2_map_pass_bit_exact_vs_oracle(config2):
    net, truth, obs = config2
    cfg = sg.SamplerConfig(same_m=M, minibatch_size=CASES, num_passes=1, map_estimate=True, seed=300)
    cpts, trace = sg.run(net, sg.DeviceSource(obs, CASES, CASES), cfg)
    onet, _ = O.koller()
    dense = obs[:, :CASES].cpu().numpy().astype(np.int32)
    res = O.run(onet, dense, same_m=M, minibatch_size=CASES, num_passes=1, map_estimate=True, seed=300)
    for a, b in zip(cpts.tables, res.cpts):
        np.testing.assert_array_equal(a, b)
    assert trace.records[0].vars_sampled == 5 * CASES * M


def test_config2_fast_mode_properties(config2):
    from paper_1511_06416_b200.engine import Engine

    net, truth, obs = config2
    cfg = sg.SamplerConfig(same_m=M, minibatch_size=CASES, num_passes=1, map_estimate=True, seed=300, rng="fast")
    eng = Engine(net, cfg)
    src = sg.DeviceSource(obs, CASES, CASES)
    mb = next(iter(src))
    eng.visit(mb, 0, M)
    torch.cuda.synchronize()
    counts = eng.prev_counts[0].cpu().numpy()
    for v in range(net.num_vars):
        a, b = eng.pack.layout.cpt_off[v], eng.pack.layout.cpt_off[v + 1]
        assert counts[a:b].sum() == M * CASES
    st = eng.lane_states(0)[:, :, :CASES]
    lat = (st < 0)
    o = obs[:, :CASES]
    # observed cells hold the data in every replica; latent flags follow the mask
    assert bool(((o >= 0).unsqueeze(1) == ~lat).all())
    assert bool(((st & 0x7F) == o.clamp(min=0).unsqueeze(1))[~lat].all())
    # numpy-mode tallies from the same CPTs agree within noise
    cfg2 = sg.SamplerConfig(same_m=M, minibatch_size=CASES, num_passes=1, map_estimate=True, seed=300)
    eng2 = Engine(net, cfg2)
    eng2.visit(mb, 0, M)
    torch.cuda.synchronize()
    c2 = eng2.prev_counts[0].cpu().numpy().astype(np.float64)
    c1 = counts.astype(np.float64)
    tot = M * CASES
    # binomial noise per cell: sd <= sqrt(tot * p(1-p)) <= 1600 (plus replica correlation, m=10)
    assert np.abs(c1 - c2).max() < 6 * np.sqrt(tot * 0.25) * np.sqrt(M)

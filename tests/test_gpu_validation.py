"""Bad input never reaches a kernel as an index (reference sampler.py:429-430:
out-of-range states raise ValidationError before any state is touched).

Host inputs are checked on the host; device-resident and pinned blocks are
checked on the device, where an out-of-range observation is written as state
0 and flagged in the error word (k_init_states, k_small_scatter), so no table
index is ever formed from it; run() raises ValidationError at the end of the
pass."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

sg = pytest.importorskip("paper_1511_06416_b200")


def _bad_obs(koller, cases=4096):
    net, truth = koller
    obs = sg.forward_sample_device(net, truth, cases, seed=1, hide_fraction=0.5, mask_seed=2)
    obs[0, 17] = 5     # difficulty is binary
    obs[3, cases - 96] = 3   # grade has 3 states: 3 is out of range
    return obs


@pytest.mark.parametrize("rng", ["numpy", "fast", "joint"])
def test_device_source_out_of_range_raises(koller, rng):
    net, _ = koller
    obs = _bad_obs(koller)
    cfg = sg.SamplerConfig(same_m=3, minibatch_size=1024, num_passes=1, seed=1, rng=rng)
    with pytest.raises(sg.ValidationError):
        sg.run(net, sg.DeviceSource(obs, 4096, 1024), cfg)


@pytest.mark.parametrize("rng", ["numpy", "fast"])
def test_host_source_out_of_range_raises(koller, rng):
    net, _ = koller
    obs = _bad_obs(koller).cpu()
    cfg = sg.SamplerConfig(same_m=2, minibatch_size=1024, num_passes=1, seed=1, rng=rng)
    with pytest.raises(sg.ValidationError):
        sg.run(net, sg.HostSource.from_dense(obs[:, :4096], 1024), cfg)
    with pytest.raises(sg.ValidationError):
        sg.HostSource.from_dense(np.full((5, 10), 200), 8)


def test_host_inputs_rejected_before_upload(koller):
    net, _ = koller
    dense = np.zeros((5, 40), dtype=np.int32)
    dense[4, 3] = 2
    with pytest.raises(sg.ValidationError):
        sg.run(net, sg.DataMatrix.from_dense(dense), sg.SamplerConfig(minibatch_size=16))
    int8 = np.zeros((5, 40), dtype=np.int8)
    int8[1, 0] = 9
    from paper_1511_06416_b200.engine import Engine

    eng = Engine(net, sg.SamplerConfig(minibatch_size=40))
    mb = sg.Minibatch(index=0, values=int8, weights=np.ones(40), num_real=40)
    with pytest.raises(sg.ValidationError):
        eng.visit(mb, 0, 1)
    with pytest.raises(sg.ValidationError):
        sg.tally_counts(net, np.full((5, 3), 2), np.ones(3))
    with pytest.raises(sg.ValidationError):
        sg.tally_counts(net, np.full((5, 3), -1), np.ones(3))


def test_sweep_rejects_out_of_range_batch(koller):
    net, truth = koller
    dense = np.zeros((5, 8), dtype=np.int32)
    dense[2, :] = -1
    batch = sg.replicate_minibatch(sg.pad_block(0, dense, 8), 2)
    batch.values[0, 1] = 7
    col = sg.color_graph(sg.moralize(net))
    with pytest.raises(sg.ValidationError):
        sg.sweep(net, col, truth, batch, 1)


def test_clean_run_after_rejection(koller):
    """The engine state is usable after a rejected block (no corrupted neighbours)."""
    net, truth = koller
    obs = sg.forward_sample_device(net, truth, 2048, seed=3, hide_fraction=0.5, mask_seed=4)
    cfg = sg.SamplerConfig(same_m=2, minibatch_size=1024, num_passes=2, seed=1, map_estimate=True)
    a, _ = sg.run(net, sg.DeviceSource(obs, 2048, 1024), cfg)
    with pytest.raises(sg.ValidationError):
        sg.run(net, sg.DeviceSource(_bad_obs(koller, 2048), 2048, 1024), cfg)
    b, _ = sg.run(net, sg.DeviceSource(obs, 2048, 1024), cfg)
    for x, y in zip(a.tables, b.tables):
        assert np.array_equal(x, y)
        assert torch.isfinite(torch.from_numpy(x)).all()

"""Pin the CPU oracle to the reference: every fixture in tests/golden/ was
produced by running the reference (tests/golden/make_golden.py); the oracle
must reproduce each one bit for bit (statistical runs excepted)."""

import numpy as np
import pytest

import oracle as O
from golden_io import RUNS_MAP, SWEEPS, edges, load, per_var, tables


def _net(d):
    return O.make_net([int(c) for c in d["cards"]], edges(d))


@pytest.mark.parametrize("name", SWEEPS)
def test_sweep_matches_reference(name):
    d = load(f"sweep_{name}")
    net = _net(d)
    cpts = tables(d, "cpt")
    values = d["before"].copy()
    missing = per_var(d, "missing", net.n)
    groups = O.greedy_coloring(net)
    flat = [v for g in groups for v in g]
    assert flat == list(d["groups"])
    counts = O.sweep(net, groups, cpts, values, missing, d["weights"], int(d["sweep_seed"]))
    np.testing.assert_array_equal(values, d["after"])
    for a, b in zip(counts, tables(d, "counts")):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("name", SWEEPS)
def test_sweep_injected_uniforms(name):
    """Injected-uniform mode: feeding the recorded uniforms reproduces the sweep."""
    d = load(f"sweep_{name}")
    net = _net(d)
    values = d["before"].copy()
    missing = per_var(d, "missing", net.n)
    inj = O.InjectedUniforms(per_var(d, "u", net.n))
    O.sweep(net, O.greedy_coloring(net), tables(d, "cpt"), values, missing, d["weights"], 0, inj)
    np.testing.assert_array_equal(values, d["after"])


def test_init_latent_matches_reference():
    d = load("init_koller")
    net, _ = O.koller()
    values, missing = O.replicate(d["dense"], int(d["m"]))
    O.init_latent(net, values, missing, int(d["seed"]), *[int(x) for x in d["context"]])
    np.testing.assert_array_equal(values, d["values"])


@pytest.mark.parametrize("name", RUNS_MAP)
def test_map_run_matches_reference(name):
    d = load(f"run_{name}")
    net, truth = O.koller()
    cfgs = {
        "map_moving": dict(same_m=2, minibatch_size=100, num_passes=3, map_estimate=True, seed=4),
        "map_exp": dict(same_m=3, minibatch_size=128, num_passes=2, map_estimate=True, seed=5,
                        accumulator_mode="exponential", exp_decay=0.7),
        "map_sweeps2": dict(same_m=[(1, 1), (2, 2)], minibatch_size=150, num_passes=3, map_estimate=True,
                            seed=6, sweeps_per_minibatch=2),
    }
    res = O.run(net, d["dense"], truth=truth, **cfgs[name])
    for a, b in zip(res.cpts, tables(d, "cpt")):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(res.kl, d["kl"])
    np.testing.assert_array_equal(res.vars_sampled, d["vars_sampled"])


def test_sampled_run_matches_reference_exactly():
    """The oracle uses numpy's own gamma sampler, so even sampled runs are exact."""
    d = load("run_sampled")
    net, truth = O.koller()
    res = O.run(net, d["dense"], same_m=5, minibatch_size=200, num_passes=20, seed=7, truth=truth)
    for a, b in zip(res.cpts, tables(d, "cpt")):
        np.testing.assert_array_equal(a, b)


def test_data_generation_matches_reference():
    d = load("data_koller")
    net, truth = O.koller()
    full = O.forward_sample(net, truth, 300, 100)
    np.testing.assert_array_equal(full, d["full"])
    np.testing.assert_array_equal(O.mask_dense(full, 0.5, 200), d["masked"])


def test_rng_sites_match_reference():
    d = load("rng")
    for i in range(len(d["seeds"])):
        seed = int(d["seeds"][i])
        label = str(d["labels"][i])
        idx = [int(x) for x in str(d["idx"][i]).split(",")]
        np.testing.assert_array_equal(O.site_key(seed, label, *idx), d["keys"][i])
        np.testing.assert_array_equal(O.site_rng(seed, label, *idx).random(17), d["draws"][i])


def test_mean_cpts_and_tally_match_reference():
    d = load("model")
    net = _net(d)
    out = O.mean_cpts(tables(d, "counts"), list(d["alphas"]))
    for a, b in zip(out, tables(d, "mean")):
        np.testing.assert_array_equal(a, b)
    tab = O.tally(net, d["tally_values"], d["tally_weights"])
    for a, b in zip(tab, tables(d, "tally")):
        np.testing.assert_array_equal(a, b)

"""GPU parity: the CUDA path against the reference-generated fixtures and the
oracle, through the package API (which calls the C-ABI library).

Bar: bit-exact states, counts and MAP CPTs (integer / index work and fp64
computed in the reference's rounding order).  Sampled Dirichlet CPTs are
checked statistically (see test_gpu_stats.py).
"""

import os

import numpy as np
import pytest

import oracle as O
from golden_io import RUNS_MAP, SWEEPS, edges, load, per_var, tables

pytestmark = pytest.mark.gpu

sg = pytest.importorskip("paper_1511_06416_b200")


def _net(d):
    return sg.build_network([int(c) for c in d["cards"]], edges(d))


def _batch(d, n):
    return sg.ReplicatedBatch(m=int(d["m"]), base_size=int(d["base_size"]), values=d["before"].copy(),
                              lane_weights=d["weights"].copy(), missing_lanes=per_var(d, "missing", n))


@pytest.mark.parametrize("name", SWEEPS)
def test_sweep_bit_exact_numpy_rng(name):
    d = load(f"sweep_{name}")
    net = _net(d)
    batch = _batch(d, net.num_vars)
    counts = sg.sweep(net, sg.color_graph(sg.moralize(net)), sg.CptSet(tables(d, "cpt")), batch,
                      int(d["sweep_seed"]))
    np.testing.assert_array_equal(batch.values, d["after"])
    for a, b in zip(counts.tables, tables(d, "counts")):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("name", SWEEPS)
def test_sweep_bit_exact_injected_uniforms(name):
    from paper_1511_06416_b200.sampler import sweep_injected

    d = load(f"sweep_{name}")
    net = _net(d)
    batch = _batch(d, net.num_vars)
    counts = sweep_injected(net, sg.color_graph(sg.moralize(net)), sg.CptSet(tables(d, "cpt")), batch,
                            per_var(d, "u", net.num_vars))
    np.testing.assert_array_equal(batch.values, d["after"])
    for a, b in zip(counts.tables, tables(d, "counts")):
        np.testing.assert_array_equal(a, b)


def test_gibbs_pass_leaves_counts_alone_and_matches():
    d = load("sweep_koller_m3")
    net = _net(d)
    batch = _batch(d, net.num_vars)
    sg.gibbs_pass(net, sg.color_graph(sg.moralize(net)), sg.CptSet(tables(d, "cpt")), batch,
                  int(d["sweep_seed"]))
    np.testing.assert_array_equal(batch.values, d["after"])


def test_init_latent_bit_exact():
    d = load("init_koller")
    from paper_1511_06416_b200.io import bundled_network_path, load_network_file

    net, _ = load_network_file(bundled_network_path("koller"))
    mb = sg.pad_block(0, d["dense"].astype(np.int32), d["dense"].shape[1])
    batch = sg.replicate_minibatch(mb, int(d["m"]))
    sg.init_latent(net, batch, int(d["seed"]), *[int(x) for x in d["context"]])
    np.testing.assert_array_equal(batch.values, d["values"])


@pytest.mark.parametrize("name", RUNS_MAP)
def test_map_run_bit_exact(name, koller):
    d = load(f"run_{name}")
    net, truth = koller
    cfgs = {
        "map_moving": sg.SamplerConfig(same_m=2, minibatch_size=100, num_passes=3, map_estimate=True, seed=4),
        "map_exp": sg.SamplerConfig(same_m=3, minibatch_size=128, num_passes=2, map_estimate=True, seed=5,
                                    accumulator_mode="exponential", exp_decay=0.7),
        "map_sweeps2": sg.SamplerConfig(same_m=[(1, 1), (2, 2)], minibatch_size=150, num_passes=3,
                                        map_estimate=True, seed=6, sweeps_per_minibatch=2),
    }
    cpts, trace = sg.run(net, sg.DataMatrix.from_dense(d["dense"]), cfgs[name], truth=truth)
    for a, b in zip(cpts.tables, tables(d, "cpt")):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal([r.kl_avg for r in trace.records], d["kl"])
    np.testing.assert_array_equal([r.vars_sampled for r in trace.records], d["vars_sampled"])


def test_forward_sample_and_mask_bit_exact(koller):
    d = load("data_koller")
    net, truth = koller
    full = sg.forward_sample(net, truth, 300, seed=100)
    np.testing.assert_array_equal(full.to_dense(), d["full"])
    dev = sg.forward_sample_device(net, truth, 300, seed=100, hide_fraction=0.5, mask_seed=200)
    np.testing.assert_array_equal(dev[:, :300].cpu().numpy().astype(np.int32), d["masked"])


def test_forward_sample_shards_compose(koller):
    """Generating cases [0, N) in two shards equals one draw (case_base offsets)."""
    net, truth = koller
    whole = sg.forward_sample_device(net, truth, 1000, seed=3, hide_fraction=0.3, mask_seed=4)[:, :1000]
    a = sg.forward_sample_device(net, truth, 400, seed=3, hide_fraction=0.3, mask_seed=4)[:, :400]
    b = sg.forward_sample_device(net, truth, 600, seed=3, hide_fraction=0.3, mask_seed=4, case_base=400)[:, :600]
    assert (whole[:, :400] == a).all() and (whole[:, 400:] == b).all()


def test_mean_cpts_and_tally_bit_exact():
    d = load("model")
    net = _net(d)
    counts = sg.CountSet([t.copy() for t in tables(d, "counts")])
    prior = sg.DirichletPrior(0.3, per_variable=tuple(float(a) for a in d["alphas"]))
    out = sg.mean_cpts(counts, prior)
    for a, b in zip(out.tables, tables(d, "mean")):
        np.testing.assert_array_equal(a, b)
    tab = sg.tally_counts(net, d["tally_values"], d["tally_weights"])
    for a, b in zip(tab.tables, tables(d, "tally")):
        np.testing.assert_array_equal(a, b)


def test_weighted_tally_matches_oracle():
    rng = np.random.default_rng(13)
    net = sg.build_network([2, 2, 2, 3, 2], [(0, 2), (0, 3), (1, 3), (3, 4)])
    onet = O.make_net([2, 2, 2, 3, 2], [(0, 2), (0, 3), (1, 3), (3, 4)])
    vals = np.stack([rng.integers(0, c, size=200) for c in net.cardinalities]).astype(np.int32)
    w = rng.random(200)
    got = sg.tally_counts(net, vals, w)
    for a, b in zip(got.tables, O.tally(onet, vals, w)):
        np.testing.assert_allclose(a, b, atol=1e-9)


def test_accumulators_bit_exact_against_oracle():
    rng = np.random.default_rng(7)
    net = sg.build_network([2, 3], [(0, 1)])
    state = sg.SamplerState(current_cpts=sg.init_cpts(net, 0), total_counts=sg.zero_counts(net))
    ref_total = [np.zeros(t.shape) for t in state.total_counts.tables]
    prev = {}
    for step in range(6):
        new = sg.CountSet([rng.integers(0, 1000, size=t.shape).astype(np.float64) for t in ref_total])
        mb = step % 2
        O.moving_sum(ref_total, None if mb not in prev else prev[mb], new.tables)
        prev[mb] = new.tables
        sg.update_moving_sum(state, mb, new)
    for a, b in zip(state.total_counts.tables, ref_total):
        np.testing.assert_array_equal(a, b)
    for step in range(5):
        new = sg.CountSet([rng.random(t.shape) * 100 for t in ref_total])
        O.exponential(ref_total, new.tables, 0.83)
        sg.update_exponential(state, new, 0.83)
    for a, b in zip(state.total_counts.tables, ref_total):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("lanes", [1, 15, 16, 17, 1000, 4099, 70001])
def test_chunked_integer_tally_bit_exact(lanes):
    """sg_tally (k_tally_chunked) vs the oracle's tally (model.py:148-165) on a
    random DAG with up to 6 parents: 16-case vector units, the ragged last
    unit, parents beyond the fourth and runs too large for a shared histogram."""
    from paper_1511_06416_b200 import netgen

    net = netgen.random_dag_network(300, max_parents=6, min_card=2, max_card=4, seed=21)
    onet = O.make_net(list(net.cardinalities), [(p, c) for c in range(net.num_vars) for p in net.parents[c]])
    rng = np.random.default_rng(lanes)
    vals = np.stack([rng.integers(0, c, size=lanes) for c in net.cardinalities]).astype(np.int32)
    w = np.ones(lanes)
    got = sg.tally_counts(net, vals, w)
    for a, b in zip(got.tables, O.tally(onet, vals, w)):
        np.testing.assert_array_equal(a, b)


def test_chunked_tally_oversized_run_bit_exact():
    """A variable whose CPT exceeds the shared histogram counts straight into
    global memory; its neighbours' runs stay on the 16-case vector path."""
    cards = [4] * 8 + [3, 2]
    edges = [(p, 7) for p in range(7)] + [(7, 8), (0, 9), (8, 9)]
    net = sg.build_network(cards, edges)
    onet = O.make_net(cards, edges)
    rng = np.random.default_rng(5)
    lanes = 50_001
    vals = np.stack([rng.integers(0, c, size=lanes) for c in cards]).astype(np.int32)
    w = np.ones(lanes)
    got = sg.tally_counts(net, vals, w)
    for a, b in zip(got.tables, O.tally(onet, vals, w)):
        np.testing.assert_array_equal(a, b)


@pytest.mark.gpu
def test_np_uniforms_equal_numpy_streams():
    """sg_np_uniforms (the numpy-parity sweep's pre-generated draws) equals
    numpy's Generator(Philox(key)).random() word for word, per variable, with
    ragged stream lengths (m * nmiss[v], not multiples of 4), an untouched
    tail, and a stream longer than its row clamped to the row."""
    import ctypes

    import torch

    from paper_1511_06416_b200 import _lib
    from paper_1511_06416_b200.sampler import DeviceBatch

    n, m, cases = 3, 3, 37
    nmiss = [0, 5, 40]  # 3 * 40 > ld: the last row is clamped to ld, nothing written past it
    db = DeviceBatch(n, m, cases, cases, torch.device("cuda"))
    db.nmiss.copy_(torch.tensor(nmiss, dtype=torch.int64))
    keys = np.array([[11, 12], [2**63 + 5, 7], [123456789, 2**40 + 3]], dtype=np.uint64)
    kd = torch.from_numpy(keys.view(np.int64)).cuda()
    ld = (m * cases + 3) // 4 * 4
    out = torch.full((n * ld + 4,), -1.0, dtype=torch.float64, device="cuda")
    off = int((-out.data_ptr() % 32) // 8)
    view = out[off:off + n * ld]
    _lib.call("sg_np_uniforms", db.ref, kd.data_ptr(), n, view.data_ptr(), ld, None)
    got = view.cpu().numpy().reshape(n, ld)
    for v in range(n):
        k = min(m * nmiss[v], ld)
        want = np.random.Generator(np.random.Philox(key=keys[v])).random(k)
        np.testing.assert_array_equal(got[v, :k], want)
        assert (got[v, k:] == -1.0).all()
    assert (out[off + n * ld:].cpu().numpy() == -1.0).all()
    if os.environ.get("SG_CHECKED_RUN") == "1":  # the checked build flags the oversized stream (and is cleared)
        assert _lib.checked_lines()["aux"] > 0

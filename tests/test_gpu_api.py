"""Behaviour of the drop-in API through the CUDA path, mirroring what the
reference's own sampler tests pin (tests/test_sampler.py of samegibbs):
run() validation and errors, zero passes, inputs never mutated, thread-count
invariance, trace bookkeeping, padding, annealing, the Trace.memory units of
both accumulator modes, and the posterior-mean limit of a fully observed run.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

sg = pytest.importorskip("paper_1511_06416_b200")


def _empirical(net, dense):
    """Count-normalised CPTs of complete data (MAP with a vanishing prior)."""
    tables = []
    for v in range(net.num_vars):
        rows, card = net.table_shape(v)
        cfg = np.zeros(dense.shape[1], dtype=np.int64)
        for p, st in zip(net.parents[v], net.parent_strides(v)):
            cfg += dense[p].astype(np.int64) * int(st)
        c = np.bincount(cfg * card + dense[v], minlength=rows * card).reshape(rows, card).astype(float)
        s = c.sum(axis=1, keepdims=True)
        tables.append(np.divide(c, s, out=np.full_like(c, 1.0 / card), where=s > 0))
    return tables


@pytest.mark.parametrize("rng", ["numpy", "fast"])
def test_fully_observed_map_is_count_normalisation(koller, rng):
    net, truth = koller
    data = sg.forward_sample(net, truth, 2000, seed=5)
    cfg = sg.SamplerConfig(minibatch_size=500, num_passes=1, map_estimate=True, prior=sg.DirichletPrior(1e-12),
                           seed=9, rng=rng)
    cpts, _ = sg.run(net, data, cfg)
    for a, b in zip(cpts.tables, _empirical(net, data.to_dense())):
        np.testing.assert_allclose(a, b, atol=1e-9)


def test_zero_passes_return_the_initial_cpts(koller):
    net, truth = koller
    data = sg.forward_sample(net, truth, 100, seed=6)
    cpts, trace = sg.run(net, data, sg.SamplerConfig(num_passes=0, minibatch_size=50, seed=77))
    for a, b in zip(cpts.tables, sg.init_cpts(net, 77).tables):
        np.testing.assert_array_equal(a, b)
    assert trace.records == []


def test_dimension_mismatch_and_empty_data_raise(koller):
    net, _ = koller
    other = sg.build_network([2, 2], [(0, 1)])
    data = sg.forward_sample(other, sg.CptSet([np.array([[0.5, 0.5]]), np.array([[0.3, 0.7], [0.6, 0.4]])]), 50,
                             seed=1)
    with pytest.raises(sg.DimensionMismatch):
        sg.run(net, data, sg.SamplerConfig(minibatch_size=10))
    empty = sg.DataMatrix(net.num_vars, 0, np.array([]), np.array([]), np.array([]))
    with pytest.raises(sg.EmptyData):
        sg.run(net, empty, sg.SamplerConfig(minibatch_size=10))


def test_out_of_range_state_raises_validation_error(koller):
    net, _ = koller
    dense = np.zeros((net.num_vars, 64), dtype=np.int32)
    dense[3, 7] = 3  # variable 3 has 3 states: 0..2
    with pytest.raises(sg.ValidationError):
        sg.run(net, sg.DataMatrix.from_dense(dense), sg.SamplerConfig(minibatch_size=32))


def test_input_matrix_is_never_mutated(koller):
    net, truth = koller
    data = sg.mask(sg.forward_sample(net, truth, 400, seed=8), 0.5, seed=9)
    snap = (data.var_idx.copy(), data.case_idx.copy(), data.values.copy())
    sg.run(net, data, sg.SamplerConfig(minibatch_size=128, num_passes=3, seed=1))
    for a, b in zip((data.var_idx, data.case_idx, data.values), snap):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("rng", ["numpy", "fast"])
def test_results_do_not_depend_on_threads(koller, rng):
    net, truth = koller
    data = sg.mask(sg.forward_sample(net, truth, 1000, seed=2), 0.5, seed=3)
    cfg = sg.SamplerConfig(minibatch_size=250, num_passes=5, same_m=2, seed=123, rng=rng)
    c1, t1 = sg.run(net, data, cfg, truth=truth, threads=1)
    c8, t8 = sg.run(net, data, cfg, truth=truth, threads=8)
    for a, b in zip(c1.tables, c8.tables):
        np.testing.assert_array_equal(a, b)
    assert [r.kl_avg for r in t1.records] == [r.kl_avg for r in t8.records]


def test_trace_records_and_annealing(koller):
    net, truth = koller
    data = sg.mask(sg.forward_sample(net, truth, 400, seed=10), 0.5, seed=11)
    cfg = sg.SamplerConfig(same_m=[(1, 2), (3, 2)], minibatch_size=100, num_passes=4, seed=6)
    _, trace = sg.run(net, data, cfg, truth=truth)
    secs = [r.seconds for r in trace.records]
    assert secs == sorted(secs)
    assert [r.pass_index for r in trace.records] == [1, 2, 3, 4]
    assert all(r.kl_avg is not None for r in trace.records)
    n = net.num_vars
    assert [r.vars_sampled for r in trace.records] == [n * 400, n * 400, n * 1200, n * 1200]


def test_padded_final_minibatch_adds_no_mass():
    net = sg.build_network([2, 2], [(0, 1)])
    truth = sg.CptSet([np.array([[0.35, 0.65]]), np.array([[0.8, 0.2], [0.25, 0.75]])])
    data = sg.forward_sample(net, truth, 450, seed=3)
    cfg = sg.SamplerConfig(minibatch_size=100, num_passes=1, map_estimate=True, prior=sg.DirichletPrior(1e-12),
                           seed=0)
    learned, _ = sg.run(net, data, cfg)
    for a, b in zip(learned.tables, _empirical(net, data.to_dense())):
        np.testing.assert_allclose(a, b, atol=1e-9)


def _model_bytes(net):
    return sum(np.zeros(net.table_shape(v)).nbytes for v in range(net.num_vars))


def test_exponential_mode_memory_keeps_no_per_minibatch_state(koller):
    net, truth = koller
    data = sg.mask(sg.forward_sample(net, truth, 600, seed=12), 0.5, seed=13)
    cfg = sg.SamplerConfig(minibatch_size=150, num_passes=3, seed=7, accumulator_mode="exponential", exp_decay=0.8)
    _, trace = sg.run(net, data, cfg)
    assert trace.memory.latent_bytes == 0
    assert trace.memory.accumulator_bytes == trace.memory.model_bytes == _model_bytes(net)


def test_moving_mode_memory_grows_only_by_bookkeeping(koller):
    net, truth = koller
    base = sg.mask(sg.forward_sample(net, truth, 400, seed=30), 0.5, seed=31)
    big = sg.replicate(base, 4)
    cfg = sg.SamplerConfig(minibatch_size=200, num_passes=2, seed=32)
    _, small = sg.run(net, base, cfg)
    _, large = sg.run(net, big, cfg)
    mb = _model_bytes(net)
    assert large.memory.accumulator_bytes - mb == 4 * (small.memory.accumulator_bytes - mb)
    assert large.memory.latent_bytes == 4 * small.memory.latent_bytes
    assert large.memory.model_bytes == small.memory.model_bytes
    assert large.memory.batch_bytes == small.memory.batch_bytes


def test_streaming_memory_is_flat_under_replication(koller):
    net, truth = koller
    base = sg.mask(sg.forward_sample(net, truth, 500, seed=14), 0.5, seed=15)
    big = sg.replicate(base, 40)
    cfg = sg.SamplerConfig(minibatch_size=250, num_passes=1, seed=8, accumulator_mode="exponential", exp_decay=0.9)
    _, a = sg.run(net, base, cfg)
    _, b = sg.run(net, big, cfg)
    assert b.memory.accumulator_bytes == a.memory.accumulator_bytes
    assert b.memory.model_bytes == a.memory.model_bytes
    assert b.memory.latent_bytes == a.memory.latent_bytes == 0
    assert b.memory.batch_bytes == a.memory.batch_bytes


@pytest.mark.parametrize("rng", ["numpy", "fast"])
def test_same_replication_shrinks_the_final_spread(rng):
    """Across-seed spread of the final CPT entries does not grow from m=1 to
    m=10 (the SAME sharpening the paper is about)."""
    net = sg.build_network([2, 2], [(0, 1)])
    truth = sg.CptSet([np.array([[0.3, 0.7]]), np.array([[0.9, 0.1], [0.2, 0.8]])])
    data = sg.mask(sg.forward_sample(net, truth, 400, seed=21), 0.5, seed=22)

    def spread(m):
        finals = []
        for seed in range(12):
            cfg = sg.SamplerConfig(same_m=m, minibatch_size=100, num_passes=10, seed=seed, rng=rng)
            cpts, _ = sg.run(net, data, cfg)
            finals.append(np.concatenate([t.ravel() for t in cpts.tables]))
        return float(np.std(np.stack(finals), axis=0).mean())

    assert spread(10) <= spread(1)


def _zero_support_problem():
    """A -> B with B = 1 impossible under every state of A: any latent A next
    to an observed B = 1 has an all-zero full conditional (sampler.py:242-244)."""
    net = sg.build_network([2, 2], [(0, 1)])
    cpts = sg.CptSet([np.array([[0.5, 0.5]]), np.array([[1.0, 0.0], [1.0, 0.0]])])
    dense = np.array([[0, -1, 1, -1], [0, 0, 0, 1]], dtype=np.int32)  # case 3: A latent, B = 1
    return net, cpts, dense


@pytest.mark.parametrize("rng", ["numpy", "fast", "joint"])
@pytest.mark.parametrize("small", [True, False])
def test_zero_support_is_flagged(rng, small):
    """sg.sweep raises ZeroSupport like the reference; the engine's kernels
    (generic and packed) set the device error word that run() turns into it."""
    from paper_1511_06416_b200 import _lib
    from paper_1511_06416_b200.engine import Engine

    net, cpts, dense = _zero_support_problem()
    if rng == "numpy" and not small:
        batch = sg.replicate_minibatch(sg.pad_block(0, dense, 4), 2)
        with pytest.raises(sg.ZeroSupport):
            sg.sweep(net, sg.color_graph(sg.moralize(net)), cpts, batch, 7)
    if rng == "numpy" and small:
        pytest.skip("the packed-lane path is FAST-mode only")
    if rng == "joint" and not small:
        pytest.skip("the joint sweep runs on packed lanes only")
    # run() starts from Dirichlet(1) CPTs (full support), so plant the degenerate
    # tables in an engine and sweep once
    eng = Engine(net, sg.SamplerConfig(same_m=2, minibatch_size=4, num_passes=1, seed=1, rng=rng), small=small)
    eng.cpt.copy_(torch.from_numpy(eng.pack.flatten(cpts.tables)))
    eng.tables_fresh = False
    eng.visit(sg.pad_block(0, dense, 4), 0, 2)
    torch.cuda.synchronize()
    assert eng.err.read() & _lib.SG_ERR_ZERO_SUPPORT


def test_no_zero_support_when_the_impossible_case_is_observed():
    """The reference raises only for latent lanes: the same CPTs with B = 1
    never next to a latent A sweep cleanly."""
    net, cpts, dense = _zero_support_problem()
    dense = dense[:, :3].copy()
    batch = sg.replicate_minibatch(sg.pad_block(0, dense, 3), 2)
    counts = sg.sweep(net, sg.color_graph(sg.moralize(net)), cpts, batch, 7)
    assert counts.tables[0].sum() == 6


def test_large_cardinality_sweep_matches_oracle():
    """Cards up to the device limit (64 states) go through the generic kernel
    bit-exactly (numpy's 8-accumulator pairwise row sums for card >= 8)."""
    import oracle as O

    rng = np.random.default_rng(8)
    cards, edges = [40, 3, 64, 5], [(0, 2), (1, 2), (2, 3)]
    net = sg.build_network(cards, edges)
    cpts = sg.CptSet([rng.dirichlet(np.full(c, 0.8), size=net.table_shape(v)[0]) for v, c in enumerate(cards)])
    dense = np.stack([rng.integers(0, c, 300) for c in cards]).astype(np.int32)
    dense[rng.random(dense.shape) < 0.5] = -1
    onet = O.make_net(cards, edges)
    values, missing = O.replicate(dense, 3)
    O.init_latent(onet, values, missing, 5, 0, 0)
    batch = sg.ReplicatedBatch(m=3, base_size=300, values=values.copy(), lane_weights=np.ones(900),
                               missing_lanes=[x.copy() for x in missing])
    counts = sg.sweep(net, sg.color_graph(sg.moralize(net)), cpts, batch, 123)
    want = O.sweep(onet, O.greedy_coloring(onet), cpts.tables, values, missing, np.ones(900), 123)
    np.testing.assert_array_equal(batch.values, values)
    for a, b in zip(counts.tables, want):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("rng", ["numpy", "fast"])
def test_all_observed_and_odd_sizes(koller, rng):
    """No latent cells: the sweep changes nothing and counts the data; minibatch
    sizes that are not multiples of 16 and a case count below the minibatch size."""
    net, truth = koller
    data = sg.forward_sample(net, truth, 37, seed=3)
    cfg = sg.SamplerConfig(same_m=3, minibatch_size=50, num_passes=1, map_estimate=True,
                           prior=sg.DirichletPrior(1e-12), seed=2, rng=rng)
    cpts, trace = sg.run(net, data, cfg)
    for a, b in zip(cpts.tables, _empirical(net, data.to_dense())):
        np.testing.assert_allclose(a, b, atol=1e-9)
    assert trace.records[0].vars_sampled == net.num_vars * 37 * 3

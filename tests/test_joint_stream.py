"""CPU checks of the joint-sweep restatement (tests/fast_stream.py) and of the
host-side joint plan (netpack.joint_plan).

The joint sweep replaces the per-variable draws of one sweep by one draw from
the sweep's transition kernel K.  K must be the composition of the
reference's per-variable Gibbs kernels (sampler.py:217-284), so the
posterior of the latent fields given the observed ones is stationary under
it: pi K = pi.  The alias rows quantise K to 2^-32.
"""

import itertools

import numpy as np
import pytest

import fast_stream as F
import oracle as O


def _kernel(rows):
    B = int(rows.shape[1]).bit_length() - 1
    return np.asarray([F.alias_probs(r, B) for r in rows], dtype=np.float64) / 2.0 ** 32


def _posterior(onet, cpts, P, obs_word, width, off, dep, keep):
    """Posterior over compact columns j of pattern P with the observed fields of obs_word."""
    K = len(dep)
    out = np.zeros(K)
    for j in range(K):
        S = (obs_word & keep) | int(dep[j])
        a = [(S >> off[v]) & ((1 << width[v]) - 1) for v in range(onet.n)]
        if any(a[v] >= onet.cards[v] for v in range(onet.n)):
            continue
        p = 1.0
        for v in range(onet.n):
            cfg = sum(a[q] * st for q, st in zip(onet.parents[v], onet.strides(v)))
            p *= cpts[v][cfg, a[v]]
        out[j] = p
    return out / out.sum()


def _random_net(rng):
    n = int(rng.integers(2, 5))
    cards = [int(rng.integers(2, 4)) for _ in range(n)]
    order = rng.permutation(n)
    edges = [(int(order[i]), int(order[j])) for i in range(n) for j in range(i + 1, n) if rng.random() < 0.5]
    onet = O.make_net(cards, edges)
    cpts = [rng.dirichlet(np.full(cards[v], 1.5), size=onet.rows(v)) for v in range(n)]
    return onet, cpts


@pytest.mark.parametrize("which", ["koller", 0, 1, 2, 3])
def test_posterior_is_stationary_under_the_joint_kernel(which):
    if which == "koller":
        onet, cpts = O.koller()
    else:
        onet, cpts = _random_net(np.random.default_rng(400 + which))
    order = [v for g in O.greedy_coloring(onet) for v in g]
    tabs = F.joint_tables(onet, cpts, order)
    width, off = F.lane_fields(onet.cards)
    for P, (B, keep, dep, rows) in tabs.items():
        if sum(width) > 6:
            break
        # one observed configuration per pattern: the valid word with observed fields 0
        obs_word = 0
        pi = _posterior(onet, cpts, P, obs_word, width, off, dep, keep)
        Kmat = np.zeros((len(dep), len(dep)))
        for j in range(len(dep)):
            S = (obs_word & keep) | int(dep[j])
            Kmat[j] = _kernel(rows[S:S + 1])[0]
        valid = pi > 0
        np.testing.assert_allclose((pi @ Kmat)[valid], pi[valid], atol=1e-8)
        np.testing.assert_allclose(Kmat[valid].sum(axis=1), 1.0, atol=1e-12)
        assert np.all(Kmat[valid][:, ~valid] == 0)  # never draws an invalid state


def test_joint_kernel_equals_sequential_per_variable_kernels():
    """Row S of K = the distribution of the sequential per-variable sweep from S
    (enumerated over every draw path), within the 2^-31 quantisation."""
    onet, cpts = O.koller()
    order = [v for g in O.greedy_coloring(onet) for v in g]
    tabs = F.joint_tables(onet, cpts, order)
    width, off = F.lane_fields(onet.cards)
    P = 0b11011  # every variable latent except var 2
    B, keep, dep, rows = tabs[P]
    col = {int(d): j for j, d in enumerate(dep)}
    for S in (0, 5, 17, 40):
        a0 = [(S >> off[v]) & ((1 << width[v]) - 1) for v in range(onet.n)]
        if any(a0[v] >= onet.cards[v] for v in range(onet.n)):
            continue
        want = np.zeros(len(dep))
        latent = [v for v in order if (P >> v) & 1]
        for xs in itertools.product(*(range(onet.cards[v]) for v in latent)):
            a = list(a0)
            p = 1.0
            for v, x in zip(latent, xs):
                p *= F._conditional(onet, cpts, v, a)[x]
                a[v] = x
            lat = sum(a[v] << off[v] for v in latent)
            want[col[lat]] += p
        np.testing.assert_allclose(_kernel(rows[S:S + 1])[0], want, atol=2e-9)


def test_joint_plan_header_matches_restatement(koller):
    from paper_1511_06416_b200.netpack import joint_plan, layout, small_plan

    net, _ = koller
    lay = layout(net)
    sp, _ = small_plan(net, lay)
    jp, head = joint_plan(sp, lay.cells)
    onet, cpts = O.koller()
    tabs = F.joint_tables(onet, cpts, list(sp.order)[:net.num_vars])
    NP = jp.patterns
    assert NP == 32 and jp.max_b == 6
    for P, (B, keep, dep, rows) in tabs.items():
        meta = int(head[NP + P])
        assert meta & 0xFF == B and (meta >> 8) & 0xFF == keep
        d0 = (meta >> 16) // 4
        np.testing.assert_array_equal(head[d0:d0 + len(dep)], dep)
    # rows follow the header in pattern order, 2^bits x 2^B words each
    offs = [int(head[P]) // 4 for P in range(1, NP)]
    assert offs[0] == jp.header_words and offs == sorted(offs)
    assert jp.words == jp.header_words + sum(64 * ((1 << tabs[P][0]) + 1) for P in range(1, NP))


def test_joint_plan_rejects_wide_lane_words():
    import paper_1511_06416_b200 as sg
    from paper_1511_06416_b200.netpack import joint_plan, layout, small_plan

    net = sg.build_network([4, 4, 4, 2], [(0, 1), (1, 2), (2, 3)])  # 7 lane bits
    lay = layout(net)
    plan = small_plan(net, lay)
    assert plan is not None and joint_plan(plan[0], lay.cells) is None


def test_joint_rng_needs_a_joint_plan():
    import paper_1511_06416_b200 as sg

    cfg = sg.SamplerConfig(rng="joint")
    assert cfg.rng == "joint"
    with pytest.raises(ValueError):
        sg.SamplerConfig(rng="bogus")


@pytest.mark.parametrize("B", [1, 2, 3, 5, 6])
def test_alias_rows_encode_the_quantised_masses_exactly(B):
    """alias_row (the restatement of csrc joint_alias_row): the column masses the
    entries encode are exactly w_j = C_j - C_{j-1} (C = the 2^32-scaled ceil of
    the cumulative sums), for random, sparse, single-column and uniform rows."""
    import math

    rng = np.random.default_rng(B)
    K = 1 << B
    rows = [rng.random(K), rng.random(K) ** 8, np.eye(K)[0], np.eye(K)[K - 1], np.ones(K),
            np.where(rng.random(K) < 0.5, 0.0, rng.random(K)), np.full(K, 1e-300)]
    for p in rows:
        if p.sum() == 0:
            p[0] = 1.0
        cum = F.warp_scan(np.asarray(p, dtype=np.float64))
        ent = F.alias_row(cum, B)
        sc = 4294967296.0 / float(cum[-1])

        def quant(c):
            x = c * sc
            return 4294967296 if (math.isnan(x) or x >= 4294967296.0) else math.ceil(x)

        C = [quant(float(cum[j])) if j < K - 1 else 4294967296 for j in range(K)]
        w = [C[j] - (C[j - 1] if j else 0) for j in range(K)]
        assert F.alias_probs(ent, B) == w
        assert sum(w) == 1 << 32
        assert np.all((ent & (K - 1)) < K)

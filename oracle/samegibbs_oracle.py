"""TEST INFRASTRUCTURE ONLY -- NumPy restatement of the reference hot path.

Each function cites the reference file:line (relative to
/root/reference/pkg/src/samegibbs/) whose behaviour it restates.  It is the
checker for the CUDA path and is pinned to golden vectors produced by the
reference itself (tests/golden/).  Networks are plain (cards, edges) specs so
the oracle shares no code with the product package.
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "Net", "make_net", "site_key", "site_seed", "site_rng", "moral_edges", "greedy_coloring",
    "replicate", "init_latent", "resample_variable", "gibbs_pass", "sweep", "tally", "init_cpts",
    "mean_cpts", "sample_cpts", "moving_sum", "exponential", "run", "forward_sample", "mask_dense",
    "UniformRecorder", "InjectedUniforms", "NumpyUniforms", "koller", "ZeroSupportError",
]


class ZeroSupportError(Exception):
    """Mirror of samegibbs.errors.ZeroSupport (errors.py:51-56)."""


# ------------------------------------------------------------------ structure

@dataclass
class Net:
    cards: list
    parents: list          # ascending (network.py:122)
    children: list         # ascending (network.py:123)
    topo: list

    @property
    def n(self) -> int:
        return len(self.cards)

    def strides(self, v) -> list:
        """Mixed radix, first parent most significant (network.py:42-48)."""
        out, acc = [], 1
        for p in reversed(self.parents[v]):
            out.append(acc)
            acc *= self.cards[p]
        return out[::-1]

    def rows(self, v) -> int:
        r = 1
        for p in self.parents[v]:
            r *= self.cards[p]
        return r


def make_net(cards, edges) -> Net:
    """Parents/children sorted, smallest-index-first Kahn order (network.py:80-124)."""
    n = len(cards)
    par = [set() for _ in range(n)]
    kid = [set() for _ in range(n)]
    for p, c in edges:
        par[c].add(int(p))
        kid[p].add(int(c))
    indeg = [len(x) for x in par]
    ready = sorted(i for i in range(n) if indeg[i] == 0)
    topo = []
    while ready:
        v = ready.pop(0)
        topo.append(v)
        for c in sorted(kid[v]):
            indeg[c] -= 1
            if indeg[c] == 0:
                ready.append(c)
        ready.sort()
    return Net([int(k) for k in cards], [sorted(x) for x in par], [sorted(x) for x in kid], topo)


def moral_edges(net: Net) -> set:
    """network.py:134-144."""
    e = set()
    for c in range(net.n):
        ps = net.parents[c]
        for i, p in enumerate(ps):
            e.add((min(p, c), max(p, c)))
            for q in ps[i + 1:]:
                e.add((p, q))
    return e


def greedy_coloring(net: Net) -> list:
    """Balanced greedy colouring (network.py:147-180); returns the groups."""
    adj = [[] for _ in range(net.n)]
    for a, b in moral_edges(net):
        adj[a].append(b)
        adj[b].append(a)
    order = sorted(range(net.n), key=lambda v: (-len(adj[v]), v))
    col = [-1] * net.n
    sizes = []
    for v in order:
        blocked = {col[u] for u in adj[v] if col[u] >= 0}
        feas = [k for k in range(len(sizes)) if k not in blocked]
        k = min(feas, key=lambda k: (sizes[k], k)) if feas else len(sizes)
        if k == len(sizes):
            sizes.append(0)
        col[v] = k
        sizes[k] += 1
    groups = [[] for _ in sizes]
    for v, k in enumerate(col):
        groups[k].append(v)
    return groups


def koller():
    """The bundled student network (data/koller.json)."""
    cards = [2, 2, 2, 3, 2]
    edges = [(0, 2), (0, 3), (1, 3), (3, 4)]
    cpts = [np.array([[0.7, 0.3]]), np.array([[0.6, 0.4]]), np.array([[0.95, 0.05], [0.2, 0.8]]),
            np.array([[0.3, 0.4, 0.3], [0.05, 0.25, 0.7], [0.9, 0.08, 0.02], [0.5, 0.3, 0.2]]),
            np.array([[0.1, 0.9], [0.4, 0.6], [0.99, 0.01]])]
    return make_net(cards, edges), cpts


# ------------------------------------------------------------------ RNG sites

def site_key(seed, label, *idx) -> np.ndarray:
    """rng.py:16-20: blake2b-128 of "seed:label:i..." as two LE uint64."""
    text = ":".join([str(int(seed)), label] + [str(int(i)) for i in idx]).encode()
    return np.frombuffer(hashlib.blake2b(text, digest_size=16).digest(), dtype="<u8").copy()


def site_seed(seed, label, *idx) -> int:
    """rng.py:28-30."""
    return int(site_key(seed, label, *idx)[0])


def site_rng(seed, label, *idx) -> np.random.Generator:
    """rng.py:23-25."""
    return np.random.Generator(np.random.Philox(key=site_key(seed, label, *idx)))


class NumpyUniforms:
    """The reference's uniform source: substream(sweep_seed, "var", v).random(k)."""

    def __call__(self, sweep_seed, v, k):
        return site_rng(sweep_seed, "var", v).random(k)


class UniformRecorder(NumpyUniforms):
    """Same stream, also records what each variable consumed (for injection tests)."""

    def __init__(self):
        self.log = {}

    def __call__(self, sweep_seed, v, k):
        u = super().__call__(sweep_seed, v, k)
        self.log[v] = u.copy()
        return u


class InjectedUniforms:
    """Caller-supplied uniforms per variable, in reference lane order."""

    def __init__(self, per_var):
        self.per_var = per_var

    def __call__(self, sweep_seed, v, k):
        u = np.asarray(self.per_var[v], dtype=np.float64)
        assert u.size == k
        return u


# ------------------------------------------------------------------ sweep

def replicate(dense_block, m):
    """sampler.py:174-187: tile m times; latent lanes = value < 0 (ascending)."""
    values = np.tile(np.asarray(dense_block, dtype=np.int32), (1, m))
    missing = [np.flatnonzero(values[v] < 0) for v in range(values.shape[0])]
    return values, missing


def init_latent(net: Net, values, missing, seed, *context):
    """sampler.py:205-214."""
    for v in range(net.n):
        lanes = missing[v]
        if lanes.size:
            values[v, lanes] = site_rng(seed, "latent_init", *context, v).integers(
                0, net.cards[v], size=lanes.size, dtype=np.int32)


def resample_variable(net: Net, tables, values, v, lanes, sweep_seed, uniforms):
    """sampler.py:217-248 (weights: parent row, then children ascending)."""
    card = net.cards[v]
    cfg = np.zeros(lanes.size, dtype=np.int64)
    for p, st in zip(net.parents[v], net.strides(v)):
        cfg += values[p, lanes].astype(np.int64) * st
    w = tables[v][cfg]
    for c in net.children[v]:
        cs = net.strides(c)
        vst = cs[net.parents[c].index(v)]
        xc = values[c, lanes]
        cfg0 = np.zeros(lanes.size, dtype=np.int64)
        for p, st in zip(net.parents[c], cs):
            if p != v:
                cfg0 += values[p, lanes].astype(np.int64) * st
        for s in range(card):
            w[:, s] *= tables[c][cfg0 + s * vst, xc]
    norm = w.sum(axis=1)
    if np.any(norm <= 0.0):
        raise ZeroSupportError(f"variable {v}")
    u = uniforms(sweep_seed, v, lanes.size)
    cum = np.cumsum(w, axis=1)
    x = (u[:, None] * norm[:, None] > cum).sum(axis=1)
    values[v, lanes] = np.minimum(x, card - 1)


def gibbs_pass(net: Net, groups, tables, values, missing, sweep_seed, uniforms=None):
    """sampler.py:251-284 (sequential order inside a group is result-neutral)."""
    uniforms = uniforms or NumpyUniforms()
    for grp in groups:
        for v in grp:
            if missing[v].size:
                resample_variable(net, tables, values, v, missing[v], sweep_seed, uniforms)


def tally(net: Net, values, weights):
    """model.py:148-165: bincount of cfg*card + x weighted by lane weight."""
    out = []
    for v in range(net.n):
        card = net.cards[v]
        cfg = np.zeros(values.shape[1], dtype=np.int64)
        for p, st in zip(net.parents[v], net.strides(v)):
            cfg += values[p].astype(np.int64) * st
        out.append(np.bincount(cfg * card + values[v], weights=weights,
                               minlength=net.rows(v) * card).reshape(net.rows(v), card))
    return out


def sweep(net: Net, groups, tables, values, missing, weights, sweep_seed, uniforms=None):
    """sampler.py:287-304."""
    gibbs_pass(net, groups, tables, values, missing, sweep_seed, uniforms)
    return tally(net, values, weights)


# ------------------------------------------------------------------ model

def init_cpts(net: Net, seed):
    """model.py:111-118."""
    return [site_rng(seed, "init_cpts", v).dirichlet(np.ones(net.cards[v]), size=net.rows(v))
            for v in range(net.n)]


def mean_cpts(total, alphas):
    """model.py:188-194."""
    out = []
    for t, a in zip(total, alphas):
        sh = t + a
        out.append(sh / sh.sum(axis=1, keepdims=True))
    return out


def sample_cpts(total, alphas, seed):
    """model.py:168-185."""
    out = []
    for i, (t, a) in enumerate(zip(total, alphas)):
        rng = site_rng(seed, "sample_cpts", i)
        params = t + a
        g = rng.standard_gamma(params)
        sums = g.sum(axis=1)
        for r in np.flatnonzero(sums <= 0.0):
            g[r] = rng.dirichlet(params[r])
            sums[r] = g[r].sum()
        out.append(g / sums[:, None])
    return out


def moving_sum(total, prev, new):
    """sampler.py:337-343 via CountSet.add (model.py:56-58)."""
    for i in range(len(total)):
        if prev is not None:
            total[i] += -1.0 * prev[i]
        total[i] += 1.0 * new[i]


def exponential(total, new, decay):
    """sampler.py:346-351 via CountSet.scale/add (model.py:56-62)."""
    for i in range(len(total)):
        total[i] *= decay
        total[i] += 1.0 * new[i]


# ------------------------------------------------------------------ driver

@dataclass
class RunResult:
    cpts: list
    kl: list = field(default_factory=list)
    vars_sampled: list = field(default_factory=list)
    seconds: list = field(default_factory=list)


def _anneal(same_m, p):
    if isinstance(same_m, int):
        return same_m
    end = 0
    for m, k in same_m:
        end += k
        if p < end:
            return m
    return same_m[-1][0]


def _kl(truth, est):
    tot, rows = 0.0, 0
    for p, q in zip(truth, est):
        keep = (p > 0) & (q > 0)
        with np.errstate(divide="ignore", invalid="ignore"):
            tot += float(np.where(keep, p * np.log(p / q), 0.0).sum())
        rows += p.shape[0]
    return tot / rows


def run(net: Net, dense, *, same_m=1, minibatch_size=1024, num_passes=1, alpha=1.0,
        accumulator_mode="moving_sum", exp_decay=1.0, sweeps_per_minibatch=1, map_estimate=False, seed=0,
        truth=None, uniforms=None, max_minibatches=None):
    """sampler.py:385-495 over a dense (n, cases) int matrix with -1 = missing."""
    import time

    dense = np.asarray(dense)
    cases = dense.shape[1]
    groups = greedy_coloring(net)
    cur = init_cpts(net, seed)
    total = [np.zeros((net.rows(v), net.cards[v])) for v in range(net.n)]
    alphas = [alpha] * net.n if np.isscalar(alpha) else list(alpha)
    per_mb, latent = {}, {}
    res = RunResult(cpts=cur)
    nmb = math.ceil(cases / minibatch_size)
    if max_minibatches is not None:
        nmb = min(nmb, max_minibatches)
    for p in range(num_passes):
        t0 = time.perf_counter()
        m = _anneal(same_m, p)
        for i in range(nmb):
            lo, hi = i * minibatch_size, min((i + 1) * minibatch_size, cases)
            block = dense[:, lo:hi].astype(np.int32)
            real = hi - lo
            if real < minibatch_size:  # pad_block sampler.py:163-171
                block = np.concatenate([block, np.full((net.n, minibatch_size - real), -1, np.int32)], axis=1)
            w = np.zeros(minibatch_size)
            w[:real] = 1.0
            values, missing = replicate(block, m)
            weights = np.tile(w, m)
            kept = latent.get(i)
            if kept is not None and all(k.size == missing[v].size for v, k in enumerate(kept)):
                for v, k in enumerate(kept):
                    values[v, missing[v]] = k
            else:
                init_latent(net, values, missing, seed, p, i)
            counts = None
            for s in range(sweeps_per_minibatch):
                counts = sweep(net, groups, cur, values, missing, weights, site_seed(seed, "sweep", p, i, s),
                               uniforms)
            if accumulator_mode == "moving_sum":
                moving_sum(total, per_mb.get(i), counts)
                per_mb[i] = counts
                latent[i] = [values[v, missing[v]].copy() for v in range(net.n)]
            else:
                exponential(total, counts, exp_decay)
            if map_estimate:
                cur = mean_cpts(total, alphas)
            else:
                cur = sample_cpts(total, alphas, site_seed(seed, "cpt_update", p, i))
        res.seconds.append(time.perf_counter() - t0)
        res.vars_sampled.append(net.n * min(cases, nmb * minibatch_size) * m * sweeps_per_minibatch)
        if truth is not None:
            res.kl.append(_kl(truth, cur))
    res.cpts = cur
    return res


# ------------------------------------------------------------------ data

def forward_sample(net: Net, cpts, num_cases, seed):
    """datagen.py:91-107, dense (n, cases) int32."""
    dense = np.zeros((net.n, num_cases), dtype=np.int32)
    for v in net.topo:
        cfg = np.zeros(num_cases, dtype=np.int64)
        for p, st in zip(net.parents[v], net.strides(v)):
            cfg += dense[p].astype(np.int64) * st
        u = site_rng(seed, "forward_sample", v).random(num_cases)
        cum = np.cumsum(cpts[v][cfg], axis=1)
        dense[v] = np.minimum((u[:, None] > cum).sum(axis=1), net.cards[v] - 1)
    return dense


def mask_dense(dense, hide, seed):
    """datagen.py:110-121 for a fully present matrix: entries in case-major order."""
    n, cases = dense.shape
    keep = site_rng(seed, "mask").random(n * cases) >= hide
    out = dense.copy()
    out[~keep.reshape(cases, n).T] = -1
    return out

"""CPT / count containers and the model-sized steps of the path.

Containers (``CptSet``, ``CountSet``, ``DirichletPrior``) keep the reference's
shape convention (``samegibbs/model.py:22-88``): one dense fp64
``(parent configs, card)`` table per variable.  The compute functions of the
path run on the device through the C-ABI:

* :func:`tally_counts` -> ``sg_tally`` / ``sg_tally_weighted`` (model.py:148-165)
* :func:`mean_cpts`    -> ``sg_mean_cpts`` (model.py:188-194), bit-exact
* :func:`sample_cpts`  -> ``sg_sample_cpts`` (model.py:179-185), statistical parity

:func:`init_cpts` is the one-time Dirichlet(1) initialisation; it runs on the
host through numpy's generator because the bit-exact contract with the
reference includes the initial CPTs (model.py:111-118) and numpy's gamma
sampler is not reproduced on the device.  :func:`full_conditional` and
:func:`accumulate_counts` are the reference's scalar helpers (test oracles of
the vectorised path), kept for API compatibility.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ShapeMismatch, ZeroSupport
from .network import Network
from .rng import derive_seed, substream

ROW_SUM_TOL = 1e-9


@dataclass(eq=False)
class CptSet:
    """Per-variable conditional probability tables."""

    tables: list[np.ndarray]

    def copy(self) -> "CptSet":
        return CptSet([np.array(t, copy=True) for t in self.tables])

    @property
    def num_rows(self) -> int:
        return sum(t.shape[0] for t in self.tables)

    def iter_rows(self):
        for t in self.tables:
            yield from t

    def validate(self) -> None:
        for i, t in enumerate(self.tables):
            if (t < 0).any() or (t > 1).any():
                raise ValueError(f"table {i} has entries outside [0, 1]")
            if np.abs(t.sum(axis=1) - 1.0).max() > ROW_SUM_TOL:
                raise ValueError(f"table {i} has a row not summing to 1")


@dataclass(eq=False)
class CountSet:
    """State counts, congruent with a CptSet."""

    tables: list[np.ndarray]

    def copy(self) -> "CountSet":
        return CountSet([np.array(t, copy=True) for t in self.tables])

    def add(self, other: "CountSet", scale: float = 1.0) -> None:
        for mine, theirs in zip(self.tables, other.tables):
            mine += scale * theirs

    def scale(self, factor: float) -> None:
        for t in self.tables:
            t *= factor

    def total_mass(self, v: int) -> float:
        return float(self.tables[v].sum())

    @property
    def nbytes(self) -> int:
        return sum(t.nbytes for t in self.tables)


@dataclass(frozen=True)
class DirichletPrior:
    """Symmetric concentration with optional per-variable overrides."""

    alpha: float = 1.0
    per_variable: tuple[float, ...] | None = None

    def __post_init__(self) -> None:
        if self.alpha <= 0:
            raise ValueError(f"alpha must be > 0, got {self.alpha}")
        if self.per_variable is not None and min(self.per_variable, default=1.0) <= 0:
            raise ValueError("per-variable alpha overrides must all be > 0")

    def alpha_for(self, v: int) -> float:
        return self.alpha if self.per_variable is None else self.per_variable[v]

    def vector(self, n: int) -> np.ndarray:
        return np.array([self.alpha_for(v) for v in range(n)], dtype=np.float64)


def zero_counts(net: Network) -> CountSet:
    return CountSet([np.zeros(net.table_shape(v)) for v in range(net.num_vars)])


def check_congruent(a, b) -> None:
    sa = [t.shape for t in a.tables]
    sb = [t.shape for t in b.tables]
    if sa != sb:
        raise ShapeMismatch(f"table shapes differ: {sa} vs {sb}")


def parent_config_index(net: Network, v: int, assignment) -> int:
    strides = net.parent_strides(v)
    return int(sum(int(assignment[p]) * int(strides[j]) for j, p in enumerate(net.parents[v])))


def init_cpts(net: Network, seed: int) -> CptSet:
    """Dirichlet(1) rows from the ``(seed, "init_cpts", v)`` streams (model.py:111-118)."""
    out = []
    for v in range(net.num_vars):
        rows, card = net.table_shape(v)
        out.append(substream(seed, "init_cpts", v).dirichlet(np.ones(card), size=rows))
    return CptSet(out)


def full_conditional(net: Network, cpts: CptSet, v: int, assignment) -> np.ndarray:
    """Scalar full conditional of v (model.py:121-139)."""
    card = net.cardinalities[v]
    a = np.array(assignment, dtype=np.int64, copy=True)
    w = np.array(cpts.tables[v][parent_config_index(net, v, a)], dtype=np.float64, copy=True)
    for s in range(card):
        a[v] = s
        for c in net.children[v]:
            w[s] *= cpts.tables[c][parent_config_index(net, c, a), a[c]]
    tot = w.sum()
    if tot <= 0.0:
        raise ZeroSupport(f"all full-conditional weights of variable {v} are zero")
    return w / tot


def accumulate_counts(net: Network, assignment, out: CountSet, weight: float = 1.0) -> None:
    """Scalar tally of one complete assignment (model.py:142-145)."""
    for v in range(net.num_vars):
        out.tables[v][parent_config_index(net, v, assignment), int(assignment[v])] += weight


# ---------------------------------------------------------------- device ops

def tally_counts(net: Network, values, weights) -> CountSet:
    """Count tables of complete assignments ``values`` (n, lanes), per-lane weights.

    0/1 weights (the engine's case) are tallied exactly in integers; other
    weights use fp64 atomics (agreement to ~1e-12, the reference's own test
    uses 1e-9, test_model.py:211-223).
    """
    from .device import device, netpack, stream_handle
    from .sampler import _upload_lanes

    dev = device()
    pack = netpack(net)
    vals = np.asarray(values)
    w = np.asarray(weights, dtype=np.float64)
    if vals.ndim != 2 or vals.shape[0] != net.num_vars or w.shape != (vals.shape[1],):
        raise ShapeMismatch("values must be (num_vars, lanes) with one weight per lane")
    lanes = vals.shape[1]
    batch = _upload_lanes(vals, None, m=1, cases=lanes, num_real=lanes, dev=dev, cards=net.cardinalities)
    binary = bool(np.all((w == 0.0) | (w == 1.0)))
    if binary and np.all(w[:int(w.sum())] == 1.0):  # a prefix of ones: plain integer tally
        batch.struct.num_real = int(w.sum())
        counts = torch.zeros(pack.cells, dtype=torch.int64, device=dev)
        _lib.call("sg_tally", pack.ref, batch.ref, counts.data_ptr(), stream_handle())
        flat = counts.cpu().numpy().astype(np.float64)
    else:
        wd = torch.from_numpy(np.ascontiguousarray(w)).to(dev)
        counts = torch.zeros(pack.cells, dtype=torch.float64, device=dev)
        _lib.call("sg_tally_weighted", pack.ref, batch.ref, wd.data_ptr(), counts.data_ptr(), stream_handle())
        flat = counts.cpu().numpy()
    return CountSet(pack.split(flat))


def _alpha_dev(prior: DirichletPrior, n: int, dev) -> torch.Tensor:
    return torch.from_numpy(prior.vector(n)).to(dev)


def mean_cpts(counts: CountSet, prior: DirichletPrior, net: Network | None = None) -> CptSet:
    """Posterior-mean rows, bit-exact with model.py:188-194."""
    from .device import device, stream_handle

    dev = device()
    pack = _pack_for_tables(counts.tables, net)
    total = torch.from_numpy(pack.flatten(counts.tables)).to(dev)
    out = torch.empty_like(total)
    _lib.call("sg_mean_cpts", pack.ref, total.data_ptr(), _alpha_dev(prior, pack.n, dev).data_ptr(),
              out.data_ptr(), stream_handle())
    return CptSet(pack.split(out.cpu().numpy()))


def sample_cpts(counts: CountSet, prior: DirichletPrior, seed: int, net: Network | None = None) -> CptSet:
    """Rows ~ Dirichlet(counts + alpha) (model.py:179-185); key derive_seed(seed, "sample_cpts")."""
    from .device import device, stream_handle

    dev = device()
    pack = _pack_for_tables(counts.tables, net)
    total = torch.from_numpy(pack.flatten(counts.tables)).to(dev)
    out = torch.empty_like(total)
    _lib.call("sg_sample_cpts", pack.ref, total.data_ptr(), _alpha_dev(prior, pack.n, dev).data_ptr(),
              derive_seed(seed, "sample_cpts"), None, out.data_ptr(), stream_handle())
    return CptSet(pack.split(out.cpu().numpy()))


def _pack_for_tables(tables, net: Network | None):
    """Row-layout pack for mean/sample: only (rows, card) shapes matter."""
    from .device import device, netpack
    from .netpack import TablePack

    if net is not None:
        return netpack(net)
    return TablePack.get(tuple((int(t.shape[0]), int(t.shape[1])) for t in tables), device())

"""The sampler API of the reference, backed by the CUDA path.

Drop-in for ``samegibbs.sampler`` (``sampler.py:51-495``): same names, same
argument meaning, same exceptions.  What changes is where the work runs:

* ``run`` keeps the whole minibatch step on the device -- replication and
  latent init (``sg_init_states``), conditional tables (``sg_build_tables``),
  the fused sweep + tally (``sg_sweep``), the accumulator (``sg_accumulate``)
  and the CPT update (``sg_mean_cpts`` / ``sg_sample_cpts``); CPTs come back
  to the host once per pass for the trace.
* ``sweep`` / ``gibbs_pass`` / ``init_latent`` accept the reference's host
  ``ReplicatedBatch``, run one device step and write ``batch.values`` back in
  place, bit-identical to the reference (numpy RNG mode).

RNG modes (``SamplerConfig.rng``):

* ``"numpy"`` (default): every uniform is the one numpy would hand the
  reference for the same site, so sweeps, tallies and MAP runs reproduce the
  reference bit for bit;
* ``"fast"``: Philox4x32-10 with (case, variable, replica) counters --
  statistically equivalent, independent of tiling and GPU count;
* ``"joint"``: small networks only (packed lane word of <= 6 bits): each
  lane's whole colour-ordered sweep is ONE draw from the sweep's transition
  kernel (the product of the full conditionals gibbs_pass draws from, in
  colour order), one Philox4x32 uniform per lane -- the same Markov chain as
  ``"fast"`` with fewer random numbers and table lookups; the throughput
  mode of the Koller configurations.

``threads`` is accepted for compatibility and, as in the reference, does not
change results (the device decides its own parallelism).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import Iterator, Sequence, Union

import numpy as np
import torch

from . import _lib
from .datagen import DataMatrix
from .device import ErrorWord, device, netpack, stream_handle
from .errors import (DimensionMismatch, EmptyData, ShapeMismatch, ValidationError, ZeroSupport,
                     DeviceError)
from .model import CountSet, CptSet, DirichletPrior, init_cpts, zero_counts
from .network import Coloring, Network, color_graph, moralize
from .rng import derive_seed

MSchedule = Union[int, Sequence[tuple[int, int]]]

ACCUMULATOR_MODES = ("moving_sum", "exponential")
RNG_MODES = ("numpy", "fast", "joint")


@dataclass
class SamplerConfig:
    """Run configuration (``sampler.py:51-87``) plus the device RNG mode."""

    same_m: MSchedule = 1
    minibatch_size: int = 1024
    num_passes: int = 1
    prior: DirichletPrior = DirichletPrior(1.0)
    accumulator_mode: str = "moving_sum"
    exp_decay: float = 1.0
    sweeps_per_minibatch: int = 1
    map_estimate: bool = False
    seed: int = 0
    rng: str = "numpy"

    def __post_init__(self) -> None:
        if isinstance(self.same_m, Sequence):
            sched = tuple((int(m), int(p)) for m, p in self.same_m)
            if not sched:
                raise ValueError("same_m schedule must be nonempty")
            if any(m < 1 or p < 1 for m, p in sched):
                raise ValueError("same_m schedule entries must have m >= 1 and passes >= 1")
            self.same_m = sched
        elif self.same_m < 1:
            raise ValueError(f"same_m must be >= 1, got {self.same_m}")
        if self.minibatch_size < 1:
            raise ValueError(f"minibatch_size must be >= 1, got {self.minibatch_size}")
        if self.num_passes < 0:
            raise ValueError(f"num_passes must be >= 0, got {self.num_passes}")
        if self.accumulator_mode not in ACCUMULATOR_MODES:
            raise ValueError(f"accumulator_mode must be one of {ACCUMULATOR_MODES}")
        if not 0.0 < self.exp_decay <= 1.0:
            raise ValueError(f"exp_decay must be in (0, 1], got {self.exp_decay}")
        if self.sweeps_per_minibatch < 1:
            raise ValueError(f"sweeps_per_minibatch must be >= 1, got {self.sweeps_per_minibatch}")
        if self.rng not in RNG_MODES:
            raise ValueError(f"rng must be one of {RNG_MODES}")


def anneal_m(schedule: MSchedule, pass_index: int) -> int:
    """Replication factor of a 0-based pass (``sampler.py:90-105``)."""
    if pass_index < 0:
        raise ValueError(f"pass_index must be >= 0, got {pass_index}")
    if isinstance(schedule, int):
        if schedule < 1:
            raise ValueError(f"m must be >= 1, got {schedule}")
        return schedule
    if not schedule:
        raise ValueError("schedule must be nonempty")
    end = 0
    for m, passes in schedule:
        end += passes
        if pass_index < end:
            return m
    return schedule[-1][0]


@dataclass(eq=False)
class Minibatch:
    """Dense block of cases; -1 = missing, weight 0 = padding (``sampler.py:108-119``).

    ``values`` is a host int array (num_vars, size) or a CUDA int8 tensor
    (device-resident sources).
    """

    index: int
    values: object
    weights: np.ndarray
    num_real: int

    @property
    def size(self) -> int:
        return int(self.values.shape[1])


@dataclass(eq=False)
class ReplicatedBatch:
    """m lane copies of a minibatch (``sampler.py:122-138``); lane r*size + c."""

    m: int
    base_size: int
    values: np.ndarray
    lane_weights: np.ndarray
    missing_lanes: list[np.ndarray]

    @property
    def num_lanes(self) -> int:
        return self.values.shape[1]


def num_minibatches(num_cases: int, minibatch_size: int) -> int:
    return math.ceil(num_cases / minibatch_size)


def pad_block(index: int, block: np.ndarray, size: int) -> Minibatch:
    """Pad a short final block with missing cells of weight 0 (``sampler.py:163-171``)."""
    real = block.shape[1]
    if real < size:
        block = np.concatenate([block, np.full((block.shape[0], size - real), -1, dtype=np.int32)], axis=1)
    weights = np.zeros(size, dtype=np.float64)
    weights[:real] = 1.0
    return Minibatch(index=index, values=block, weights=weights, num_real=real)


class MatrixSource:
    """Re-iterable minibatches of an in-memory DataMatrix (``sampler.py:141-156``)."""

    def __init__(self, data: DataMatrix, minibatch_size: int):
        self.num_vars = data.num_vars
        self.num_cases = data.num_cases
        self.minibatch_size = minibatch_size
        self._data = data

    def __iter__(self) -> Iterator[Minibatch]:
        b = self.minibatch_size
        for i in range(num_minibatches(self.num_cases, b)):
            lo, hi = i * b, min((i + 1) * b, self.num_cases)
            yield pad_block(i, self._data.dense_block(lo, hi), b)


def as_source(data, minibatch_size: int):
    if isinstance(data, DataMatrix):
        return MatrixSource(data, minibatch_size)
    return data


def replicate_minibatch(mb: Minibatch, m: int) -> ReplicatedBatch:
    """Host replication for callers of the batch-level API (``sampler.py:174-187``)."""
    if m < 1:
        raise ValueError(f"m must be >= 1, got {m}")
    vals = mb.values
    if isinstance(vals, torch.Tensor):
        vals = vals.cpu().numpy()
    values = np.tile(np.asarray(vals), (1, m)).astype(np.int32)
    return ReplicatedBatch(m=m, base_size=mb.size, values=values,
                           lane_weights=np.tile(np.asarray(mb.weights, dtype=np.float64), m),
                           missing_lanes=[np.flatnonzero(values[v] < 0) for v in range(values.shape[0])])


# ----------------------------------------------------------------- device batch

def _pitch(cases: int) -> int:
    return max(16, (cases + 15) // 16 * 16)


class DeviceBatch:
    """A replicated minibatch resident in HBM (``sg_batch``)."""

    def __init__(self, n: int, m: int, cases: int, num_real: int, dev: torch.device,
                 case_base: int = 0, states: torch.Tensor | None = None):
        self.n, self.m, self.cases, self.num_real = n, m, cases, num_real
        self.pitch = _pitch(cases)
        self.dev = dev
        self.states = states if states is not None else torch.empty((n, m, self.pitch), dtype=torch.int8,
                                                                    device=dev)
        self.obs = None
        self.rank = None
        self.nmiss = torch.zeros(n, dtype=torch.int64, device=dev)
        s = _lib.SgBatch()
        s.states = self.states.data_ptr()
        s.m, s.cases, s.pitch, s.num_real = m, cases, self.pitch, num_real
        s.case_base = case_base
        s.nmiss = self.nmiss.data_ptr()
        self.struct = s
        self.ref = __import__("ctypes").byref(s)

    def set_latent_hint(self, fraction: float) -> None:
        """Latent share of the batch's cells (kernel choice for large networks, sg_batch.latent_permille)."""
        self.struct.latent_permille = int(round(1000 * min(1.0, max(0.0, float(fraction)))))

    def set_obs(self, obs: torch.Tensor) -> None:
        """Attach the (n, pitch) int8 observation block the ranks refer to."""
        self.obs = obs

    def compute_nmiss(self) -> None:
        """Latent case counts per variable only (no rank array)."""
        nblk = max(1, (self.cases + 4095) // 4096)
        scratch = torch.empty(self.n * nblk, dtype=torch.int64, device=self.dev)
        _lib.call("sg_rank_latent", self.n, self.obs.data_ptr(), self.obs.stride(0), self.cases, None, 0,
                  self.nmiss.data_ptr(), scratch.data_ptr(), stream_handle())
        self._scratch = scratch

    def nmiss_total(self) -> int:
        return int(self.nmiss.sum().item())

    def compute_ranks(self) -> None:
        if self.rank is None:
            self.rank = torch.empty((self.n, self.pitch), dtype=torch.int32, device=self.dev)
            self.struct.rank = self.rank.data_ptr()
            self.struct.ld_rank = self.pitch
        nblk = max(1, (self.cases + 4095) // 4096)
        scratch = torch.empty(self.n * nblk, dtype=torch.int64, device=self.dev)
        _lib.call("sg_rank_latent", self.n, self.obs.data_ptr(), self.obs.stride(0), self.cases,
                  self.rank.data_ptr(), self.pitch, self.nmiss.data_ptr(), scratch.data_ptr(), stream_handle())
        self._scratch = scratch  # keep alive until the stream has consumed it


def _obs_from_values(vals_rep0: np.ndarray, latent: np.ndarray, pitch: int, dev) -> torch.Tensor:
    n, cases = vals_rep0.shape
    obs = np.zeros((n, pitch), dtype=np.int8)
    v8 = vals_rep0.astype(np.int64)
    if cases and (v8.max(initial=0) > 127):
        raise ValueError("states above 127 are not supported by the int8 lane layout")
    obs[:, :cases] = np.where(latent, -1, v8).astype(np.int8)
    return torch.from_numpy(obs).to(dev)


def _upload_lanes(values: np.ndarray, missing_lanes, m: int, cases: int, num_real: int, dev,
                  cards=None) -> DeviceBatch:
    """Host (n, m*cases) int values + latent lane lists -> DeviceBatch (flags in bit 7).

    ``cards``: per-variable cardinalities; every cell must hold a state below
    its card (checked here, before any device index is formed)."""
    vals = np.asarray(values)
    n = vals.shape[0]
    if vals.shape[1] != m * cases:
        raise ShapeMismatch("values must have m * base_size lanes")
    db = DeviceBatch(n, m, cases, num_real, dev)
    lat = np.zeros((n, m * cases), dtype=bool)
    if missing_lanes is not None:
        for v, lanes in enumerate(missing_lanes):
            lat[v, np.asarray(lanes, dtype=np.int64)] = True
    db.set_latent_hint(lat.mean() if lat.size else 0.0)
    st = np.zeros((n, m, db.pitch), dtype=np.int8)
    if (vals < 0).any() and missing_lanes is not None:
        # the reference samples cells listed in missing_lanes; any other cell must hold a state
        if (vals[~lat] < 0).any():
            raise ValidationError("a non-latent cell holds no state")
    if missing_lanes is None and (vals < 0).any():
        raise ValidationError("values must be complete assignments (a cell holds no state)")
    if cards is not None and vals.size:
        top = np.asarray(cards, dtype=np.int64)[:, None]
        if (vals >= top).any():
            raise ValidationError("data contains a state >= its variable's cardinality")
    cell = np.where(vals < 0, 0, vals).astype(np.int64)
    if cell.size and cell.max() > 127:
        raise ValueError("states above 127 are not supported by the int8 lane layout")
    packed = (cell | (lat.astype(np.int64) << 7)).astype(np.uint8).view(np.int8)
    st[:, :, :cases] = packed.reshape(n, m, cases)
    db.states.copy_(torch.from_numpy(st))
    if missing_lanes is not None:
        lat3 = lat.reshape(n, m, cases)
        if m > 1 and not (lat3 == lat3[:, :1, :]).all():
            raise ValidationError("latent lanes differ between replicas (not a SAME batch)")
        db.set_obs(_obs_from_values(np.where(lat3[:, 0, :], -1, cell.reshape(n, m, cases)[:, 0, :]),
                                    lat3[:, 0, :], db.pitch, dev))
    return db


def _var_keys(seed: int, label: str, context: tuple, n: int, dev) -> torch.Tensor:
    from .device import var_keys

    return var_keys(None, seed, label, context, n)


def _download_states(db: DeviceBatch, batch: ReplicatedBatch) -> None:
    st = db.states[:, :, :db.cases].cpu().numpy().astype(np.int32) & 0x7F
    batch.values[...] = st.reshape(db.n, db.m * db.cases)


def _batch_num_real(batch: ReplicatedBatch) -> int | None:
    """num_real if lane weights are the pad_block pattern (ones then zeros per replica)."""
    w = np.asarray(batch.lane_weights, dtype=np.float64).reshape(batch.m, batch.base_size)
    real = int((w[0] == 1.0).sum())
    pattern = np.zeros(batch.base_size)
    pattern[:real] = 1.0
    if np.array_equal(w, np.broadcast_to(pattern, w.shape)):
        return real
    return None


def _raise_errors(word: int) -> None:
    if word & _lib.SG_ERR_ZERO_SUPPORT:
        raise ZeroSupport("all full-conditional weights of some latent cell are zero")
    if word & _lib.SG_ERR_STATE_RANGE:
        raise ValidationError("data contains a state >= its variable's cardinality")
    if word & _lib.SG_ERR_REJECT_OVERFLOW:
        raise DeviceError("too many Lemire rejections in a latent-init stream")


def _device_pass(net: Network, coloring: Coloring, cpts: CptSet, batch: ReplicatedBatch, sweep_seed: int,
                 tally: bool, uniforms=None, rng: str = "numpy") -> CountSet | None:
    """One device sweep over a host batch.  ``uniforms``: optional per-variable
    fp64 arrays in reference lane order (injected-uniform mode)."""
    dev = device()
    pack = netpack(net, coloring)
    n = net.num_vars
    num_real = _batch_num_real(batch) if tally else batch.base_size
    db = _upload_lanes(batch.values, batch.missing_lanes, batch.m, batch.base_size,
                       num_real if num_real is not None else batch.base_size, dev, net.cardinalities)
    db.compute_ranks()
    cpt = torch.from_numpy(pack.flatten(cpts.tables)).to(dev)
    ptab = torch.empty(max(1, pack.layout.scalars["ptab_size"]), dtype=torch.float64, device=dev)
    ftab = torch.empty(pack.layout.scalars["ftab_size"] + 1, dtype=torch.int32, device=dev)
    s = stream_handle()
    _lib.call("sg_build_tables", pack.ref, cpt.data_ptr(), ptab.data_ptr(), ftab.data_ptr(), s)
    err = ErrorWord(dev)
    counts = None
    if tally and num_real is not None:
        counts = torch.zeros(pack.cells, dtype=torch.int64, device=dev)
    cptr = None if counts is None else counts.data_ptr()
    if uniforms is not None:
        sizes = [len(batch.missing_lanes[v]) for v in range(n)]
        for v in range(n):
            if len(uniforms[v]) != sizes[v]:
                raise ShapeMismatch(f"variable {v} needs {sizes[v]} uniforms, got {len(uniforms[v])}")
        flat = np.concatenate([np.asarray(uniforms[v], dtype=np.float64) for v in range(n)] + [np.zeros(1)])
        off = np.zeros(n, dtype=np.int64)
        off[1:] = np.cumsum(sizes)[:-1]
        u_dev = torch.from_numpy(flat).to(dev)
        off_dev = torch.from_numpy(off).to(dev)
        _lib.call("sg_sweep", pack.ref, db.ref, cpt.data_ptr(), ptab.data_ptr(), ftab.data_ptr(),
                  _lib.SG_RNG_INJECTED, 0, None, None, u_dev.data_ptr(), off_dev.data_ptr(), cptr, err.ptr, s)
    elif rng == "fast":
        _lib.call("sg_sweep", pack.ref, db.ref, cpt.data_ptr(), ptab.data_ptr(), ftab.data_ptr(),
                  _lib.SG_RNG_FAST, int(sweep_seed) & 0xFFFFFFFFFFFFFFFF, None, None, None, None, cptr, err.ptr, s)
    else:
        keys = _var_keys(sweep_seed, "var", (), n, dev)
        _lib.call("sg_sweep", pack.ref, db.ref, cpt.data_ptr(), ptab.data_ptr(), ftab.data_ptr(),
                  _lib.SG_RNG_NUMPY, 0, None, keys.data_ptr(), None, None, cptr, err.ptr, s)
    word = err.read()
    _raise_errors(word)
    _download_states(db, batch)
    if not tally:
        return None
    if counts is not None:
        return CountSet(pack.split(counts.cpu().numpy().astype(np.float64)))
    # general lane weights: weighted tally of the post-sweep states
    from .model import tally_counts
    return tally_counts(net, batch.values, batch.lane_weights)


def gibbs_pass(net: Network, coloring: Coloring, cpts: CptSet, batch: ReplicatedBatch, sweep_seed: int,
               executor=None, cache=None) -> None:
    """One chromatic sweep over every latent cell, in place (``sampler.py:251-284``)."""
    _device_pass(net, coloring, cpts, batch, sweep_seed, tally=False)


def sweep(net: Network, coloring: Coloring, cpts: CptSet, batch: ReplicatedBatch, sweep_seed: int,
          executor=None, cache=None) -> CountSet:
    """Sweep + tally of the final assignments (``sampler.py:287-304``)."""
    return _device_pass(net, coloring, cpts, batch, sweep_seed, tally=True)


def sweep_injected(net: Network, coloring: Coloring, cpts: CptSet, batch: ReplicatedBatch,
                   uniforms) -> CountSet:
    """Sweep with caller-supplied uniforms: ``uniforms[v]`` holds one fp64 per
    latent lane of v, in the order the reference consumes them
    (``batch.missing_lanes[v]`` ascending, sampler.py:245)."""
    return _device_pass(net, coloring, cpts, batch, 0, tally=True, uniforms=uniforms)


def sweep_fast(net: Network, coloring: Coloring, cpts: CptSet, batch: ReplicatedBatch, key: int) -> CountSet:
    """Sweep in the fast RNG mode (Philox4x32-10 keyed by ``key``)."""
    return _device_pass(net, coloring, cpts, batch, key, tally=True, rng="fast")


def init_latent(net: Network, batch: ReplicatedBatch, seed: int, *context: int) -> None:
    """Uniform initial states of every latent cell (``sampler.py:205-214``), bit-exact."""
    dev = device()
    pack = netpack(net)
    n = net.num_vars
    db = _upload_lanes(batch.values, batch.missing_lanes, batch.m, batch.base_size, batch.base_size, dev,
                       net.cardinalities)
    db.compute_ranks()
    keys = _var_keys(seed, "latent_init", tuple(context), n, dev)
    rej = torch.empty(n * (_lib.REJ_SLACK + 2), dtype=torch.int64, device=dev)
    err = ErrorWord(dev)
    _lib.call("sg_init_states", pack.ref, db.ref, db.obs.data_ptr(), db.pitch, _lib.SG_RNG_NUMPY, 0,
              keys.data_ptr(), rej.data_ptr(), err.ptr, stream_handle())
    _raise_errors(err.read())
    _download_states(db, batch)


# ----------------------------------------------------------------- accumulators

@dataclass(eq=False)
class SamplerState:
    """Engine state between visits (``sampler.py:307-334``)."""

    current_cpts: CptSet
    total_counts: CountSet
    per_minibatch_counts: dict = field(default_factory=dict)
    latent: dict = field(default_factory=dict)
    pass_index: int = 0
    minibatch_index: int = 0
    batch: ReplicatedBatch | None = None

    def check_moving_sum(self, rel_tol: float = 1e-6) -> None:
        for i, total in enumerate(self.total_counts.tables):
            acc = np.zeros_like(total)
            for counts in self.per_minibatch_counts.values():
                acc += counts.tables[i]
            scale = max(float(acc.max(initial=0.0)), 1.0)
            if np.abs(acc - total).max(initial=0.0) > rel_tol * scale:
                raise AssertionError(f"moving sum out of sync on variable {i}")


def _accumulate_host(total: CountSet, new: CountSet, prev: CountSet | None, mode: int, decay: float) -> None:
    """Run sg_accumulate_f64 over host CountSets and write the result back."""
    from .netpack import TablePack

    dev = device()
    shapes = tuple((int(t.shape[0]), int(t.shape[1])) for t in total.tables)
    pack = TablePack.get(shapes, dev)
    t = torch.from_numpy(pack.flatten(total.tables)).to(dev)
    nw = torch.from_numpy(pack.flatten(new.tables)).to(dev)
    pv = torch.from_numpy(pack.flatten(prev.tables)).to(dev) if prev is not None else None
    _lib.call("sg_accumulate_f64", mode, t.data_ptr(), nw.data_ptr(), None if pv is None else pv.data_ptr(),
              decay, pack.cells, stream_handle())
    out = pack.split(t.cpu().numpy())
    for mine, res in zip(total.tables, out):
        mine[...] = res


def update_moving_sum(state: SamplerState, mb_id: int, new_counts: CountSet) -> None:
    """Swap minibatch mb_id's contribution in the running total (``sampler.py:337-343``)."""
    prev = state.per_minibatch_counts.get(mb_id)
    _accumulate_host(state.total_counts, new_counts, prev, _lib.SG_ACC_MOVING, 1.0)
    state.per_minibatch_counts[mb_id] = new_counts


def update_exponential(state: SamplerState, new_counts: CountSet, decay: float) -> None:
    """Decayed running sum (``sampler.py:346-351``)."""
    if not 0.0 < decay <= 1.0:
        raise ValueError(f"decay must be in (0, 1], got {decay}")
    _accumulate_host(state.total_counts, new_counts, None, _lib.SG_ACC_EXPONENTIAL, decay)


# ----------------------------------------------------------------- trace

@dataclass
class TraceRecord:
    pass_index: int
    seconds: float
    kl_avg: float | None
    vars_per_sec: float | None
    vars_sampled: int


@dataclass
class MemoryStats:
    """Byte accounting in the reference's units (fp64 tables, int32 latents,
    ``sampler.py:363-370``); ``device_bytes`` is what the engine holds in HBM."""

    model_bytes: int = 0
    accumulator_bytes: int = 0
    latent_bytes: int = 0
    batch_bytes: int = 0
    device_bytes: int = 0


@dataclass
class Trace:
    records: list[TraceRecord] = field(default_factory=list)
    memory: MemoryStats = field(default_factory=MemoryStats)


def run(net: Network, data, cfg: SamplerConfig, truth: CptSet | None = None, threads: int = 1,
        engine_hook=None) -> tuple[CptSet, Trace]:
    """Train CPTs on a minibatch stream (``sampler.py:385-495``) on the device."""
    from .engine import Engine

    source = as_source(data, cfg.minibatch_size)
    if source.num_vars != net.num_vars:
        raise DimensionMismatch(f"data has {source.num_vars} variables, network has {net.num_vars}")
    if source.num_cases == 0:
        raise EmptyData("data stream contains no cases")
    eng = Engine(net, cfg)
    if engine_hook is not None:
        engine_hook(eng)
    return eng.run(source, truth)

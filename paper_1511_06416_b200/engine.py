"""Device-resident SAME engine: the body of ``run()`` (reference sampler.py:385-495).

Per minibatch visit everything stays on the GPU and on one stream:

    obs upload (or device view)          sg_rank_latent (numpy RNG only)
    sg_init_states | restore latents     sg_build_tables(current CPTs)
    sg_sweep x S (tally on the last)     sg_accumulate
    sg_mean_cpts | sg_sample_cpts        -> CPTs for the next visit

The host only hashes a few site keys per visit and reads the error word, the
CPTs and the trace once per pass.  Counts are exact 64-bit integers on the
device; the running total is fp64 and follows the reference's rounding.
"""

from __future__ import annotations

import time

import numpy as np
import torch

from . import _lib
from .device import ErrorWord, device, netpack, stream_handle
from .errors import ValidationError
from .metrics import kl_avg
from .model import CptSet, init_cpts
from .network import Network, color_graph, moralize
from .rng import derive_seed, stream_key_ints
from .sampler import (DeviceBatch, MemoryStats, SamplerConfig, Trace, TraceRecord, _pitch, _raise_errors,
                      anneal_m)


class PinnedRing:
    """Pinned host staging buffers reused only after their last H2D copy ran."""

    def __init__(self, shape, dtype, slots: int = 2):
        self.bufs = [torch.empty(shape, dtype=dtype, pin_memory=True) for _ in range(slots)]
        self.events = [torch.cuda.Event() for _ in range(slots)]
        self.used = [False] * slots
        self.i = 0

    def slot(self):
        i = self.i
        self.i = (i + 1) % len(self.bufs)
        if self.used[i]:
            self.events[i].synchronize()
        self.used[i] = True
        return self.bufs[i], self.events[i]


class Engine:
    def __init__(self, net: Network, cfg: SamplerConfig, case_base: int = 0, comm=None):
        self.net = net
        self.cfg = cfg
        self.dev = device()
        self.coloring = color_graph(moralize(net))
        self.pack = netpack(net, self.coloring)
        self.n = net.num_vars
        self.case_base = case_base
        self.comm = comm  # optional count all-reduce hook (multi-GPU, see parallel.py)
        lay = self.pack.layout
        cells = self.pack.cells
        d = self.dev
        self.cpt = torch.from_numpy(self.pack.flatten(init_cpts(net, cfg.seed).tables)).to(d)
        self.total = torch.zeros(cells, dtype=torch.float64, device=d)
        self.counts = torch.zeros(cells, dtype=torch.int64, device=d)
        self.ptab = torch.empty(max(1, lay.scalars["ptab_size"]), dtype=torch.float64, device=d)
        self.ftab = torch.empty(max(1, lay.scalars["ftab_size"]), dtype=torch.int32, device=d)
        self.alpha = torch.from_numpy(cfg.prior.vector(self.n)).to(d)
        self.err = ErrorWord(d)
        self.rng_mode = _lib.SG_RNG_NUMPY if cfg.rng == "numpy" else _lib.SG_RNG_FAST
        self.prev_counts: dict[int, torch.Tensor] = {}
        self.latent: dict[int, DeviceBatch] = {}   # moving-sum: resident lane states per minibatch
        self.nmiss_host: dict[int, np.ndarray] = {}
        self.keys = torch.empty((self.n, 2), dtype=torch.int64, device=d)
        self._keys_ring = PinnedRing((self.n, 2), torch.int64)
        self.rej = torch.empty(self.n * (_lib.REJ_SLACK + 2), dtype=torch.int64, device=d)
        self._obs_cache: dict[int, torch.Tensor] = {}
        self._obs_rings: dict[int, PinnedRing] = {}
        self.batch_bytes = 0
        self.sweep_events = None  # list -> (start, end, sweeps) CUDA events around each visit's sweeps

    # ------------------------------------------------------------ helpers
    def _upload_keys(self, seed: int, label: str, context: tuple) -> None:
        host, done = self._keys_ring.slot()
        kh = host.numpy().view(np.uint64)
        for v in range(self.n):
            kh[v] = stream_key_ints(seed, label, *context, v)
        self.keys.copy_(host, non_blocking=True)
        done.record()

    def _obs_for(self, mb) -> tuple[torch.Tensor, int]:
        """Device (n, pitch) int8 observation block of a minibatch."""
        vals = mb.values
        size = mb.size
        pitch = _pitch(size)
        if isinstance(vals, torch.Tensor) and vals.is_cuda:
            if vals.dtype == torch.int8 and vals.stride(1) == 1 and vals.stride(0) % 16 == 0 \
                    and vals.data_ptr() % 16 == 0:
                return vals, vals.stride(0)
            buf = torch.full((self.n, pitch), -1, dtype=torch.int8, device=self.dev)
            buf[:, :size].copy_(vals)
            return buf, pitch
        if isinstance(vals, torch.Tensor) and vals.dtype == torch.int8 and vals.is_pinned() \
                and vals.shape[1] == pitch and vals.is_contiguous():
            # host-resident pinned int8 block (streaming sources): one async H2D copy
            buf = self._obs_cache.get(pitch)
            if buf is None:
                buf = self._obs_cache[pitch] = torch.empty((self.n, pitch), dtype=torch.int8, device=self.dev)
            buf.copy_(vals, non_blocking=True)
            return buf, pitch
        host = vals.numpy() if isinstance(vals, torch.Tensor) else np.asarray(vals)
        if host.dtype != np.int8:
            cards = np.asarray(self.net.cardinalities)[:, None]
            if ((host >= cards) & (host >= 0)).any():
                raise ValidationError("data contains a state >= its variable's cardinality")
            host = host.astype(np.int8)
        buf = self._obs_cache.get(pitch)
        if buf is None:
            buf = self._obs_cache[pitch] = torch.empty((self.n, pitch), dtype=torch.int8, device=self.dev)
        ring = self._obs_rings.get(pitch)
        if ring is None:
            ring = self._obs_rings[pitch] = PinnedRing((self.n, pitch), torch.int8)
        pinned, done = ring.slot()
        pinned.numpy()[:, :size] = host
        pinned.numpy()[:, size:] = -1
        buf.copy_(pinned, non_blocking=True)
        done.record()
        return buf, pitch

    # ------------------------------------------------------------ one visit
    def visit(self, mb, pass_index: int, m: int) -> None:
        cfg = self.cfg
        s = stream_handle()
        obs, ld = self._obs_for(mb)
        size = mb.size
        stored = self.latent.get(mb.index) if cfg.accumulator_mode == "moving_sum" else None
        if stored is not None and stored.m == m and stored.cases == size:
            db = stored
            db.set_obs(obs)
        else:
            db = DeviceBatch(self.n, m, size, int(mb.num_real), self.dev, self.case_base)
            db.set_obs(obs)
        db.struct.num_real = int(mb.num_real)
        _lib.call("sg_check_range", self.pack.ref, obs.data_ptr(), ld, size, self.err.ptr, s)
        if self.rng_mode == _lib.SG_RNG_NUMPY:
            db.compute_ranks()
        elif db is not stored and cfg.accumulator_mode == "moving_sum":
            db.compute_nmiss()  # latent counts for the memory accounting only
        if db is not stored:
            if self.rng_mode == _lib.SG_RNG_NUMPY:
                self._upload_keys(cfg.seed, "latent_init", (pass_index, mb.index))
                _lib.call("sg_init_states", self.pack.ref, db.ref, obs.data_ptr(), ld, _lib.SG_RNG_NUMPY, 0,
                          self.keys.data_ptr(), self.rej.data_ptr(), self.err.ptr, s)
            else:
                key = derive_seed(cfg.seed, "latent_init", pass_index, mb.index)
                _lib.call("sg_init_states", self.pack.ref, db.ref, obs.data_ptr(), ld, _lib.SG_RNG_FAST, key,
                          None, None, self.err.ptr, s)
        _lib.call("sg_build_tables", self.pack.ref, self.cpt.data_ptr(), self.ptab.data_ptr(),
                  self.ftab.data_ptr(), s)
        new_counts = torch.zeros_like(self.counts) if cfg.accumulator_mode == "moving_sum" else self.counts
        if new_counts is self.counts:
            new_counts.zero_()
        S = cfg.sweeps_per_minibatch
        timing = self.sweep_events
        if timing is not None:
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
        for sw in range(S):
            sweep_seed = derive_seed(cfg.seed, "sweep", pass_index, mb.index, sw)
            counts_ptr = new_counts.data_ptr() if sw == S - 1 else None
            if self.rng_mode == _lib.SG_RNG_NUMPY:
                self._upload_keys(sweep_seed, "var", ())
                _lib.call("sg_sweep", self.pack.ref, db.ref, self.cpt.data_ptr(), self.ptab.data_ptr(),
                          self.ftab.data_ptr(), _lib.SG_RNG_NUMPY, 0, self.keys.data_ptr(), None, None,
                          counts_ptr, self.err.ptr, s)
            else:
                _lib.call("sg_sweep", self.pack.ref, db.ref, self.cpt.data_ptr(), self.ptab.data_ptr(),
                          self.ftab.data_ptr(), _lib.SG_RNG_FAST, sweep_seed, None, None, None, counts_ptr,
                          self.err.ptr, s)
        if timing is not None:
            ev1.record()
            timing.append((ev0, ev1, S))
        if self.comm is not None:
            self.comm(new_counts)
        if cfg.accumulator_mode == "moving_sum":
            prev = self.prev_counts.get(mb.index)
            _lib.call("sg_accumulate", _lib.SG_ACC_MOVING, self.total.data_ptr(), new_counts.data_ptr(),
                      None if prev is None else prev.data_ptr(), 1.0, self.pack.cells, s)
            self.prev_counts[mb.index] = new_counts
            self.latent[mb.index] = db
        else:
            _lib.call("sg_accumulate", _lib.SG_ACC_EXPONENTIAL, self.total.data_ptr(), new_counts.data_ptr(),
                      None, cfg.exp_decay, self.pack.cells, s)
        if cfg.map_estimate:
            _lib.call("sg_mean_cpts", self.pack.ref, self.total.data_ptr(), self.alpha.data_ptr(),
                      self.cpt.data_ptr(), s)
        else:
            key = derive_seed(derive_seed(cfg.seed, "cpt_update", pass_index, mb.index), "sample_cpts")
            _lib.call("sg_sample_cpts", self.pack.ref, self.total.data_ptr(), self.alpha.data_ptr(), key,
                      self.cpt.data_ptr(), s)
        self.batch_bytes = max(self.batch_bytes, self.n * m * size * 4 + m * size * 8)
        self._last_batch = db

    # ------------------------------------------------------------ run
    def current_cpts(self) -> CptSet:
        return CptSet(self.pack.split(self.cpt.cpu().numpy()))

    def run(self, source, truth: CptSet | None = None):
        cfg = self.cfg
        trace = Trace()
        cell_bytes = self.pack.cells * 8
        trace.memory.model_bytes = cell_bytes
        trace.memory.accumulator_bytes = cell_bytes
        torch.cuda.synchronize()
        start = time.perf_counter()
        for pass_index in range(cfg.num_passes):
            pass_start = time.perf_counter()
            m = anneal_m(cfg.same_m, pass_index)
            for mb in source:
                self.visit(mb, pass_index, m)
            word = self.err.read()  # synchronises the stream
            _raise_errors(word)
            now = time.perf_counter()
            secs = now - pass_start
            sampled = self.n * source.num_cases * m * cfg.sweeps_per_minibatch
            kl = kl_avg(truth, self.current_cpts()) if truth is not None else None
            trace.records.append(TraceRecord(pass_index=pass_index + 1, seconds=now - start, kl_avg=kl,
                                             vars_per_sec=sampled / secs if secs > 0 else None,
                                             vars_sampled=sampled))
        mem = trace.memory
        mem.accumulator_bytes = cell_bytes * (1 + len(self.prev_counts))
        latent = 0
        for db in self.latent.values():
            latent += 4 * db.m * int(db.nmiss_total())
        mem.latent_bytes = latent
        mem.batch_bytes = self.batch_bytes
        mem.model_bytes = cell_bytes
        mem.device_bytes = int(sum(t.numel() * t.element_size() for t in
                                   [self.cpt, self.total, self.counts, self.ptab, self.ftab]
                                   + list(self.prev_counts.values())
                                   + [db.states for db in self.latent.values()]))
        return self.current_cpts(), trace

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

import ctypes
import math
import time

import numpy as np
import torch

from . import _lib
from .device import ErrorWord, device, netpack, site_keys, stream_handle, var_keys
from .errors import ValidationError
from .metrics import kl_avg
from .io import pack_bits
from .model import CptSet, init_cpts
from .network import Network, color_graph, moralize
from .rng import derive_seed
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


def copy_rows(dst: torch.Tensor, src: torch.Tensor, cols: int) -> None:
    """``dst[:, :cols] = src[:, :cols]`` in stream order for device (or pinned)
    row blocks: one 2-D copy (a byte-wise strided copy kernel moved the 5 MB
    C2 block at ~0.3 TB/s)."""
    if (dst.dim() == 2 and src.dim() == 2 and dst.dtype == src.dtype and dst.stride(1) == 1 and src.stride(1) == 1
            and dst.shape[0] == src.shape[0] and (src.is_cuda or src.is_pinned())):
        es = dst.element_size()
        _lib.call("sg_copy2d_async", dst.data_ptr(), dst.stride(0) * es, src.data_ptr(), src.stride(0) * es, cols * es,
                  dst.shape[0], stream_handle())
    else:
        dst[:, :cols].copy_(src[:, :cols], non_blocking=True)


# scratch for the numpy-parity sweep's pre-generated uniforms (n * m * cases
# doubles); larger sweeps draw them inside the sweep instead
NP_UNIFORM_BUDGET = 8 << 30


class SmallBatch:
    """Packed-lane minibatch (sg_small layout): one uint8 word per lane, slots bucketed by latent pattern."""

    def __init__(self, n: int, m: int, cases: int, dev: torch.device):
        self.n, self.m, self.cases = n, m, cases
        self.lane_ld = max(4, (cases + 3) // 4 * 4)  # words per replica-quad row
        self.lanes = torch.empty(((m + 3) // 4, self.lane_ld), dtype=torch.int32, device=dev)
        self.pattern = torch.empty(max(1, cases), dtype=torch.uint8, device=dev)
        self.case_id = torch.empty(max(1, cases), dtype=torch.int32, device=dev)
        # sg_small_prepare: per-(pattern, block) bucket counts + the pattern of each case
        self.scratch = torch.empty(128 * 296 + (cases + 1) // 2 + 1, dtype=torch.int32, device=dev)
        self.nmiss = torch.zeros(n, dtype=torch.int64, device=dev)
        self.num_real = cases
        self.dev = dev

    def count_latent(self, obs: torch.Tensor, ld: int) -> None:
        nblk = max(1, (self.cases + 4095) // 4096)
        scratch = torch.empty(self.n * nblk, dtype=torch.int64, device=self.dev)
        _lib.call("sg_rank_latent", self.n, obs.data_ptr(), ld, self.cases, None, 0, self.nmiss.data_ptr(),
                  scratch.data_ptr(), stream_handle())
        self._scratch = scratch

    def nmiss_total(self) -> int:
        return int(self.nmiss.sum().item())

    @property
    def states(self) -> torch.Tensor:
        return self.lanes


class Engine:
    def __init__(self, net: Network, cfg: SamplerConfig, case_base: int = 0, comm=None,
                 small: bool | None = None, exchange=None):
        self.net = net
        self.cfg = cfg
        self.dev = device()
        self.coloring = color_graph(moralize(net))
        self.pack = netpack(net, self.coloring)
        # the pack is shared (cached per network); the large-network sweep's
        # blanket-factor scratch is this engine's own
        self.sweep_net, self._sweep_net_keep = self.pack.private_ref()
        self.n = net.num_vars
        self.case_base = case_base
        self.comm = comm  # optional count all-reduce hook (multi-GPU, see parallel.py)
        self.exchange = exchange  # NUMPY-mode sharding: global rank prefixes (parallel.rank_prefix_exchange)
        lay = self.pack.layout
        cells = self.pack.cells
        d = self.dev
        self.cpt = torch.from_numpy(self.pack.flatten(init_cpts(net, cfg.seed).tables)).to(d)
        self.total = torch.zeros(cells, dtype=torch.float64, device=d)
        self.counts = torch.zeros(cells, dtype=torch.int64, device=d)
        self.ptab = torch.empty(max(1, lay.scalars["ptab_size"]), dtype=torch.float64, device=d)
        self.ftab = torch.empty(lay.scalars["ftab_size"] + 1, dtype=torch.int32, device=d)
        self.alpha = torch.from_numpy(cfg.prior.vector(self.n)).to(d)
        self.err = ErrorWord(d)
        self.rng_mode = _lib.SG_RNG_NUMPY if cfg.rng == "numpy" else _lib.SG_RNG_FAST
        self.prev_counts: dict[int, torch.Tensor] = {}
        self.latent: dict[int, DeviceBatch] = {}   # moving-sum: resident lane states per minibatch
        self.nmiss_host: dict[int, np.ndarray] = {}
        self.keys = torch.empty((self.n, 2), dtype=torch.int64, device=d)
        self._np_uniforms = {}  # row length -> (storage, aligned view, inj_off) of numpy_sweep
        self.rej = torch.empty(self.n * (_lib.REJ_SLACK + 2), dtype=torch.int64, device=d)
        self._obs_cache: dict[int, torch.Tensor] = {}
        self._obs_rings: dict[int, PinnedRing] = {}
        self.batch_bytes = 0
        self.sweep_events = None  # list -> (start, end, sweeps) CUDA events around each visit's sweeps
        # packed-lane path: FAST RNG and a lane state that fits one byte (sg_small.cu)
        max_m = cfg.same_m if isinstance(cfg.same_m, int) else max(mm for mm, _ in cfg.same_m)
        can_small = self.rng_mode == _lib.SG_RNG_FAST and self.pack.small is not None and max_m <= 32
        self.use_small = can_small if small is None else (bool(small) and can_small)
        # joint sweep (rng="joint"): one draw per lane from the sweep's transition kernel
        self.joint = cfg.rng == "joint"
        if self.joint and (not self.use_small or self.pack.joint is None):
            raise ValueError("rng='joint' needs a network whose packed lane word has <= 6 bits "
                             "(cards <= 4, n <= 6) and same_m <= 32; use rng='fast'")
        if self.use_small:
            self.stab = torch.empty(max(1, self.pack.small.tab_words), dtype=torch.int32, device=d)
        if self.joint:
            jp = self.pack.joint
            blob = np.zeros(jp.words, dtype=np.uint32)
            blob[:jp.header_words] = self.pack.joint_header
            self.jblob = torch.from_numpy(blob.view(np.int32)).to(d)
            # full conditionals p_v(x | lane word), written by the step tail for sg_joint_tables
            self.vprob = torch.zeros(self.n * (4 << self.pack.small.bits), dtype=torch.float64, device=d)
            self.jsync = torch.zeros(4, dtype=torch.int32, device=d)  # sg_step_tail_joint's hand-off + ticket words
            # the tail slices' static preparation, built once (sg_joint_prep)
            nb = ctypes.c_int64()
            _lib.call("sg_joint_prep_bytes", self.pack.small_ref, self.pack.joint_ref, ctypes.byref(nb))
            self.jprep = torch.empty(max(16, nb.value), dtype=torch.uint8, device=d)
            _lib.call("sg_joint_prep", self.pack.ref, self.pack.small_ref, self.pack.joint_ref, self.jblob.data_ptr(),
                      self.jprep.data_ptr(), stream_handle())
        self.tables_fresh = False  # conditional tables reflect self.cpt
        self.graph_replay = True   # run(): replay steady-state visits as CUDA graphs
        self._latent_hint = None   # latent share of the first generic minibatch (sg_batch.latent_permille)

    # ------------------------------------------------------------ helpers
    def numpy_sweep(self, db, counts_ptr, s) -> None:
        """One numpy-parity sweep (keys already in ``self.keys``): the sweep's
        uniforms are generated ahead of it, four per Philox4x64 block
        (``sg_np_uniforms``), and the sweep runs in injected mode -- bit-identical
        to drawing them in the sweep (SG_RNG_NUMPY), which computes a whole block
        per uniform and is kept beyond the scratch budget."""
        ld = (db.m * db.cases + 3) // 4 * 4
        # with a rank-prefix exchange nmiss counts every rank's latent cells (its
        # streams are indexed globally): draw in the sweep
        if self.n * ld * 8 > NP_UNIFORM_BUDGET or self.exchange is not None:
            _lib.call("sg_sweep", self.sweep_net, db.ref, self.cpt.data_ptr(), self.ptab.data_ptr(),
                      self.ftab.data_ptr(), _lib.SG_RNG_NUMPY, 0, None, self.keys.data_ptr(), None, None,
                      counts_ptr, self.err.ptr, s)
            return
        buf = self._np_uniforms.get(ld)
        if buf is None:  # one buffer per row length, kept for the engine's life (graphs hold its address)
            u = torch.empty(self.n * ld + 4, dtype=torch.float64, device=self.dev)
            off = int((-u.data_ptr() % 32) // 8)  # 32-byte aligned rows
            buf = (u, u[off:off + self.n * ld],
                   torch.arange(self.n, dtype=torch.int64, device=self.dev) * ld)
            self._np_uniforms[ld] = buf
        _, uv, inj = buf
        _lib.call("sg_np_uniforms", db.ref, self.keys.data_ptr(), self.n, uv.data_ptr(), ld, s)
        _lib.call("sg_sweep", self.sweep_net, db.ref, self.cpt.data_ptr(), self.ptab.data_ptr(),
                  self.ftab.data_ptr(), _lib.SG_RNG_INJECTED, 0, None, None, uv.data_ptr(), inj.data_ptr(),
                  counts_ptr, self.err.ptr, s)

    def _upload_keys(self, seed: int, label: str, context: tuple) -> None:
        """Per-variable site keys of one sweep / latent init, hashed on the device."""
        var_keys(self.keys, seed, label, context, self.n)

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
        # host blocks of any dtype are range-checked before the upload (sampler.py:429-430);
        # device and pinned blocks are checked on the device, and an out-of-range state is
        # written as state 0 + the error bit, never used as an index
        cards = np.asarray(self.net.cardinalities)[:, None]
        if ((host >= cards) | (host < -1)).any():
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
        """One minibatch visit (sampler.py:428-471): stage, S sweeps, tally, accumulate, CPT update."""
        cfg = self.cfg
        s = stream_handle()
        obs, ld = self._obs_for(mb)
        size = mb.size
        moving = cfg.accumulator_mode == "moving_sum"
        stored = self.latent.get(mb.index) if moving else None
        if stored is not None and not (stored.m == m and stored.cases == size):
            stored = None
        if not self.use_small:  # the packed sweep checks the block in its own launch
            _lib.call("sg_check_range", self.pack.ref, obs.data_ptr(), ld, size, self.err.ptr, s)
        if self.use_small:
            db = stored if stored is not None else SmallBatch(self.n, m, size, self.dev)
            db.num_real = int(mb.num_real)
            if stored is None:
                key = derive_seed(cfg.seed, "latent_init", pass_index, mb.index)
                _lib.call("sg_small_prepare", self.pack.small_ref, obs.data_ptr(), ld, size, m, self.case_base,
                          key, 1, db.scratch.data_ptr(), db.pattern.data_ptr(), db.case_id.data_ptr(),
                          db.lanes.data_ptr(), db.lane_ld, None, s)
                if moving:
                    db.count_latent(obs, ld)
        else:
            db = stored if stored is not None else DeviceBatch(self.n, m, size, int(mb.num_real), self.dev,
                                                               self.case_base)
            if stored is None:
                if self._latent_hint is None:  # one host sync per engine: the sweep's kernel choice
                    self._latent_hint = float((obs[:, :size] < 0).float().mean())
                db.set_latent_hint(self._latent_hint)
            db.set_obs(obs)
            db.struct.num_real = int(mb.num_real)
            if self.rng_mode == _lib.SG_RNG_NUMPY:
                db.compute_ranks()
                if self.exchange is not None:  # ranks and counts over the global minibatch
                    prefix, total = self.exchange(db.nmiss)
                    db.rank += prefix.to(torch.int32)[:, None]
                    db.nmiss.copy_(total)
            elif stored is None and moving:
                db.compute_nmiss()  # latent counts for the memory accounting only
            if stored is None:
                if self.rng_mode == _lib.SG_RNG_NUMPY:
                    self._upload_keys(cfg.seed, "latent_init", (pass_index, mb.index))
                    _lib.call("sg_init_states", self.pack.ref, db.ref, obs.data_ptr(), ld, _lib.SG_RNG_NUMPY, 0,
                              self.keys.data_ptr(), self.rej.data_ptr(), self.err.ptr, s)
                else:
                    key = derive_seed(cfg.seed, "latent_init", pass_index, mb.index)
                    _lib.call("sg_init_states", self.pack.ref, db.ref, obs.data_ptr(), ld, _lib.SG_RNG_FAST, key,
                              None, None, self.err.ptr, s)
        if not self.tables_fresh:  # the previous visit's finish built them from the current CPTs
            _lib.call("sg_build_tables", self.pack.ref, self.cpt.data_ptr(), self.ptab.data_ptr(),
                      self.ftab.data_ptr(), s)
            if self.use_small:
                _lib.call("sg_small_tables", self.pack.ref, self.pack.small_ref, self.ftab.data_ptr(),
                          self.stab.data_ptr(), s)
            self.joint_tables(s, from_finish=False)
            self.tables_fresh = True
        new_counts = torch.zeros_like(self.counts) if moving else self.counts
        if not moving:
            new_counts.zero_()
        S = cfg.sweeps_per_minibatch
        timing = self.sweep_events
        if timing is not None:
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
        prev = self.prev_counts.get(mb.index) if moving else None
        key = 0 if cfg.map_estimate else derive_seed(derive_seed(cfg.seed, "cpt_update", pass_index, mb.index),
                                                     "sample_cpts")
        tail_check = self.tail_checks_obs
        f = self.finish_args(new_counts, prev, key, check=(obs.data_ptr(), ld, 8, size) if tail_check else None)
        for sw in range(S):
            sweep_seed = derive_seed(cfg.seed, "sweep", pass_index, mb.index, sw)
            last = sw == S - 1
            counts_ptr = new_counts.data_ptr() if last else None
            if self.use_small:
                if sw:
                    self.sweep_fence(s)
                self.packed_sweep(db, size, m, sweep_seed, None, counts_ptr, obs.data_ptr() if last else None, ld, s,
                                  prefetch_only=tail_check)
            elif self.rng_mode == _lib.SG_RNG_NUMPY:
                self._upload_keys(sweep_seed, "var", ())
                self.numpy_sweep(db, counts_ptr, s)
            else:
                _lib.call("sg_sweep", self.sweep_net, db.ref, self.cpt.data_ptr(), self.ptab.data_ptr(),
                          self.ftab.data_ptr(), _lib.SG_RNG_FAST, sweep_seed, None, None, None, None, counts_ptr,
                          self.err.ptr, s)
        if timing is not None:
            ev1.record()
            timing.append((ev0, ev1, S))
        if self.comm is not None:
            self.comm(new_counts)
        self.step_tail(f, s)
        if moving:
            self.prev_counts[mb.index] = new_counts
            self.latent[mb.index] = db
        self.batch_bytes = max(self.batch_bytes, self.n * m * size * 4 + m * size * 8)
        self._last_batch = db

    @property
    def tail_checks_obs(self) -> bool:
        """The joint path range-checks a visit's observation block in the step
        tail's row slices, while their preparation lands and the model update
        draws the gammas (off the sweep's critical path); with a count all-reduce
        between the two the sweep keeps the check."""
        return self.joint and self.comm is None

    def finish_args(self, new_counts, prev_counts, key: int, key_dev: int | None = None, clear=None,
                    cursor=None, cpt_host: torch.Tensor | None = None, check=None):
        """``sg_finish`` of one visit: accumulate, CPT update, next visit's tables
        (``cpt_host``: pinned host tensor the kernel also stores the new CPTs in)."""
        cfg = self.cfg
        f = _lib.SgFinish()
        f.acc_mode = _lib.SG_ACC_MOVING if cfg.accumulator_mode == "moving_sum" else _lib.SG_ACC_EXPONENTIAL
        f.map_estimate = 1 if cfg.map_estimate else 0
        f.decay = cfg.exp_decay
        f.total = self.total.data_ptr()
        f.new_counts = new_counts.data_ptr()
        f.prev_counts = None if prev_counts is None else prev_counts.data_ptr()
        f.alpha = self.alpha.data_ptr()
        f.key = key
        f.key_dev = key_dev
        f.cpt = self.cpt.data_ptr()
        f.ptab = self.ptab.data_ptr()
        f.ftab = self.ftab.data_ptr()
        f.stab = self.stab.data_ptr() if self.use_small else None
        f.clear_counts = None if clear is None else clear.data_ptr()
        # the packed sweep reads only the packed words: build them straight from the CPTs
        f.flags = _lib.SG_FINISH_PACKED_ONLY if self.use_small else 0
        f.vprob = self.vprob.data_ptr() if self.joint else None
        f.cpt_host = None if cpt_host is None else cpt_host.data_ptr()
        if check is not None:  # (observation block pointer, row bytes, bits per case, cases)
            f.check_obs, f.check_ld, f.check_bits, f.check_cases = check
            f.check_err = self.err.ptr
        if cursor is not None:
            table, index, kps, current = cursor
            f.key_table, f.key_index, f.kps, f.key_current = table.data_ptr(), index.data_ptr(), kps, current.data_ptr()
        self._finish_keepalive = f
        return f

    def packed_sweep(self, db, size: int, m: int, key: int, key_dev, counts_ptr, obs_ptr, ld: int, s,
                     obs_bits: int = 8, prefetch_only: bool = False) -> None:
        """Sweep + tally of a packed-lane minibatch: per-variable draws
        (sg_small_sweep) or, with rng="joint", one draw per lane (sg_joint_sweep;
        ``obs_bits`` 4 / 2: the range-checked block is packed, ``ld`` bytes per row)."""
        head = (db.pattern.data_ptr(), db.case_id.data_ptr(), db.lanes.data_ptr(), db.lane_ld, size, db.num_real, m,
                self.case_base, key, key_dev, self.pack.small_jcell.data_ptr(), self.pack.cells, counts_ptr,
                self.ftab.data_ptr() + 4 * self.pack.layout.scalars["ftab_size"], obs_ptr, ld)
        if self.joint:
            # prefetch_only: the step tail range-checks the block; the sweep only warms L2 for it
            bits = (obs_bits if obs_bits < 8 else 0) | (_lib.SG_OBS_PREFETCH_ONLY if prefetch_only else 0)
            _lib.call("sg_joint_sweep", self.pack.small_ref, self.pack.joint_ref, self.stab.data_ptr(),
                      self.jblob.data_ptr(), *head, bits, self.err.ptr, s)
        else:
            if obs_bits < 8:
                raise ValueError("packed observation blocks are range-checked by the joint sweep only")
            _lib.call("sg_small_sweep", self.pack.small_ref, self.stab.data_ptr(), *head, self.err.ptr, s)

    @staticmethod
    def sweep_fence(s) -> None:
        """Before the 2nd..S-th packed sweep of a visit: a plain (non-PDL) launch.
        The packed sweeps load their first slot's lane words before their PDL
        wait -- safe after the step tail, which never writes lanes, but not
        right after another sweep; an ordinary launch in between starts only
        when that sweep has completed."""
        _lib.call("sg_noop", 1, 32, 0, s)

    def step_tail(self, f, s) -> None:
        """Accumulate, CPT update and the next visit's tables: one single-CTA
        launch, or with rng="joint" one grid that also builds the joint rows."""
        if self.joint:
            _lib.call("sg_step_tail_joint", self.pack.ref, self.pack.small_ref, f, self.pack.joint_ref,
                      self.jblob.data_ptr(), self.jsync.data_ptr(), self.jprep.data_ptr(), s)
        else:
            _lib.call("sg_step_finish", self.pack.ref, self.small_ptr, f, s)

    def joint_tables(self, s, from_finish: bool = True) -> None:
        """Joint-sweep rows from the current CPTs (after every CPT update);
        ``from_finish``: the step tail has just written the conditionals."""
        if self.joint:
            _lib.call("sg_joint_tables", self.pack.ref, self.pack.small_ref, self.pack.joint_ref, self.cpt.data_ptr(),
                      self.vprob.data_ptr() if from_finish else None, self.jblob.data_ptr(), s)

    @property
    def small_ptr(self):
        return self.pack.small_ref if self.use_small else None

    def lane_states(self, mb_index: int) -> torch.Tensor:
        """int8 [n][m][pitch] lane states of a resident minibatch (generic layout, flags in bit 7)."""
        db = self.latent[mb_index] if mb_index in self.latent else self._last_batch
        if isinstance(db, SmallBatch):
            out = DeviceBatch(self.n, db.m, db.cases, db.cases, self.dev)
            _lib.call("sg_small_export", self.pack.small_ref, out.ref, db.case_id.data_ptr(), db.pattern.data_ptr(),
                      db.lanes.data_ptr(), db.lane_ld, stream_handle())
            return out.states
        return db.states

    # ------------------------------------------------------------ run
    def current_cpts(self) -> CptSet:
        return CptSet(self.pack.split(self.cpt.cpu().numpy()))

    def graphs_ok(self) -> bool:
        """Steady-state visits may be graph-replayed: moving sum (resident lanes)
        and no host collective inside the step (NCCL all-reduces are capturable)."""
        if self.cfg.accumulator_mode != "moving_sum" or not self.graph_replay:
            return False
        return self.comm is None or getattr(self.comm, "capturable", False)

    def run(self, source, truth: CptSet | None = None):
        """All passes of ``run()`` (sampler.py:385-495) without a host round trip per visit.

        The first visit of a minibatch (and the first after the SAME factor
        changes) runs eagerly and leaves its lanes resident; the following
        visits of that minibatch replay two captured step graphs
        (:class:`StepGraphs`: same kernels, same keys, bit-identical results).
        Per pass the engine records a CUDA event and, with ``truth``, a device
        snapshot of the CPTs; the host synchronises once at the end, checks
        the error word and builds the trace (pass times from the events,
        ``kl_avg`` from the snapshots in the reference's fp64 arithmetic)."""
        cfg = self.cfg
        trace = Trace()
        cell_bytes = self.pack.cells * 8
        torch.cuda.synchronize()
        start = torch.cuda.Event(enable_timing=True)
        start.record()
        marks, snaps = [], []
        snap_all = truth is not None and cfg.num_passes * cell_bytes <= (1 << 30)
        graphs: dict[int, StepGraphs] = {}
        use_graphs = self.graphs_ok()
        sched = [anneal_m(cfg.same_m, p) for p in range(cfg.num_passes)]
        # exponential accumulator on the packed / joint path: fresh visits replayed as stream graphs
        # (every full minibatch; the first visit and a padded last block run eagerly)
        full = source.num_cases // cfg.minibatch_size
        stream_ok = (cfg.accumulator_mode == "exponential" and self.use_small and self.graph_replay
                     and isinstance(cfg.same_m, int) and full >= 1
                     and (self.comm is None or getattr(self.comm, "capturable", False)))
        stream: StreamGraphs | None = None
        host_t0 = time.perf_counter()
        kls = []
        for pass_index in range(cfg.num_passes):
            m = sched[pass_index]
            end_same = pass_index
            while end_same < cfg.num_passes and sched[end_same] == m:
                end_same += 1
            for mb in source:
                if stream_ok and mb.index < full and (pass_index, mb.index) != (0, 0) and mb.size == cfg.minibatch_size:
                    if stream is None:
                        visits = [(p, i) for p in range(cfg.num_passes) for i in range(full) if (p, i) != (0, 0)]
                        stream = StreamGraphs(self, cfg.minibatch_size, m, visits)
                    stream.step(mb)
                    continue
                g = graphs.get(mb.index)
                if g is not None and (g.m != m or not g.accepts(mb)):
                    g.finish()
                    del graphs[mb.index]
                    g = None
                if g is not None:
                    g.step(mb)
                    continue
                self.visit(mb, pass_index, m)
                if use_graphs and pass_index + 1 < end_same:
                    graphs[mb.index] = StepGraphs(self, mb, m, range(pass_index + 1, end_same),
                                                  obs_buffer=StepGraphs.view_of(mb))
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            marks.append(ev)
            if truth is not None:
                if snap_all:
                    snaps.append(self.cpt.clone())
                else:  # very large models: one CPT read-back per pass
                    _raise_errors(self.err.read())
                    kls.append(kl_avg(truth, self.current_cpts()))
        for g in graphs.values():
            g.finish()
        torch.cuda.synchronize()
        host_secs = time.perf_counter() - host_t0
        _raise_errors(self.err.read())
        if snap_all and snaps:
            stacked = torch.stack(snaps).cpu().numpy()
            kls = [kl_avg(truth, CptSet(self.pack.split(row))) for row in stacked]
        prev_s = 0.0
        for pass_index, ev in enumerate(marks):
            now = start.elapsed_time(ev) * 1e-3
            secs = now - prev_s
            prev_s = now
            sampled = self.n * source.num_cases * sched[pass_index] * cfg.sweeps_per_minibatch
            trace.records.append(TraceRecord(pass_index=pass_index + 1, seconds=now,
                                             kl_avg=kls[pass_index] if truth is not None else None,
                                             vars_per_sec=sampled / secs if secs > 0 else None,
                                             vars_sampled=sampled))
        self.host_seconds = host_secs
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


class StepGraphs:
    """CUDA-graph replay of the steady-state visit of one resident minibatch.

    A moving-sum visit whose lanes are already resident (every pass after the
    first) is a fixed sequence of ~7 launches; replaying it as a graph removes
    the host's per-launch cost.  The per-visit random keys (sweep keys, the
    Dirichlet key) are precomputed for the planned passes into a device table
    that ``sg_keys_advance`` steps through at the head of each replay, and the
    new/previous count buffers alternate between two graphs.  Replays run
    exactly the kernels ``Engine.visit`` launches with exactly the same keys,
    so results equal eager visits bit for bit (every RNG mode: in numpy mode
    each replay hashes its per-variable sweep keys on the device).
    """

    def __init__(self, eng: Engine, mb, m: int, pass_indices, obs_buffer: torch.Tensor | None = None,
                 nibbles: bool = False, host_block: torch.Tensor | None = None, readback=(), obs_bits: int = 8,
                 timing: bool = False, visits_per_replay: int = 1):
        """``obs_buffer``: device int8 (n, pitch) tensor the graphs read the
        minibatch's observations from; the caller keeps it filled (e.g. a
        device-resident source).  Default: a private buffer that
        :meth:`step` refills from the minibatch passed to it.  ``obs_bits``
        4 or 2 (``nibbles=True`` = 4; joint sweep, private buffers): the
        observation blocks travel in the packed .sgb form (io.pack_bits;
        1/2 or 1/4 of the host-to-device bytes) and are range-checked in that
        form on the device.

        ``host_block`` (pinned, the private buffers' layout): every step()
        also uploads this block into the buffer of the visit after next
        (three private buffers, so each upload has two replays' time to
        land) on a copy stream (a copy engine), overlapped with the replays,
        ordered by events; with ``visits_per_replay`` 2 it may hold one block
        per visit of a replay (shape (2, ...)), uploaded with one copy.  The
        copy is asynchronous: a caller
        that refills ``host_block`` between steps must first wait for
        :attr:`upload_done` (the event of the last upload).  With the moving
        sum the replayed minibatch keeps its lanes resident, so the uploaded
        block is range-checked each visit but its observed values are the
        resident ones (the reference re-reads the same data every pass); a
        stream of different minibatches is replayed by :class:`StreamGraphs`,
        which samples each uploaded block.  ``readback``: pairs
        (device tensor, pinned host tensor) copied back at the end of each
        replay (e.g. the CPTs).  ``timing``: external timing events bracket the
        sweep node(s) inside each graph; :meth:`sweep_ms` reads the last
        replay's sweep duration (call after synchronising).
        ``visits_per_replay`` 2: each graph holds two consecutive visits (the
        second sweep's prologue overlaps the first tail under PDL, and one
        graph launch serves two visits); step() then replays two visits and
        takes no minibatch (host-fed or device-resident observations)."""
        cfg = eng.cfg
        self.vpr = int(visits_per_replay)
        if self.vpr not in (1, 2):
            raise ValueError("visits_per_replay must be 1 or 2")
        pass_indices = list(pass_indices)
        if self.vpr > 1 and (timing or len(pass_indices) % self.vpr):
            raise ValueError("two visits per replay: an even number of visits, no sweep timing")
        if cfg.accumulator_mode != "moving_sum":
            raise ValueError("graph replay of resident minibatches needs the moving-sum accumulator")
        db = eng.latent.get(mb.index)
        if db is None or db.m != m or db.cases != mb.size:
            raise ValueError("visit the minibatch once (eagerly) before capturing its graph")
        self.eng, self.mb, self.m, self.db = eng, mb, m, db
        S = cfg.sweeps_per_minibatch
        self.kps = kps = S + 1
        passes = list(pass_indices)
        table = np.empty((len(passes), kps), dtype=np.uint64)
        for i, p in enumerate(passes):
            for s in range(S):
                table[i, s] = derive_seed(cfg.seed, "sweep", p, mb.index, s)
            table[i, S] = derive_seed(derive_seed(cfg.seed, "cpt_update", p, mb.index), "sample_cpts")
        d = eng.dev
        self.table = torch.from_numpy(table.view(np.int64)).to(d)
        self.idx = torch.zeros(1, dtype=torch.int32, device=d)
        self.cur = torch.zeros(kps, dtype=torch.int64, device=d)
        self.planned = len(passes)
        self.replayed = 0
        prev = eng.prev_counts[mb.index]
        self.cbuf = [torch.zeros_like(prev), prev.clone()]
        self.obs_bits = 4 if nibbles else int(obs_bits)
        if self.obs_bits not in (8, 4, 2):
            raise ValueError("obs_bits must be 8, 4 or 2")
        self.nibbles = self.obs_bits < 8  # packed blocks (4- or 2-bit)
        if self.nibbles and (obs_buffer is not None or (eng.use_small and not eng.joint)):
            raise ValueError("packed uploads need private observation buffers and the joint or generic sweep")
        # generic sweep: a packed block is unpacked into one int8 block inside
        # the graph and range-checked there (the joint sweep reads it packed)
        self._unpacked = None
        if self.nibbles and not eng.use_small:
            self._unpacked = torch.empty((eng.n, _pitch(mb.size)), dtype=torch.int8, device=eng.dev)
        if obs_buffer is None:
            # two private buffers, one per graph parity: step(mb) uploads the next
            # visit's block on a copy stream while the current visit runs
            src, _ = eng._obs_for(mb)
            bufs = []
            shape, dt = self.obs_geometry(eng.n, mb.size, self.obs_bits)
            # host-fed graphs keep 3 x visits_per_replay: the uploads for the visits two
            # replays ahead start with the current replay, into the buffers the previous
            # replay read, so each upload has two replays' time to land
            nbuf = 3 * self.vpr if host_block is not None else 2
            # one allocation: a replay's visits own consecutive buffers, so a host
            # block per visit (host_block of shape (vpr, ...)) uploads with one copy
            whole = torch.empty((nbuf, *shape), dtype=dt, device=d)
            for i in range(nbuf):
                b = whole[i]
                if self.nibbles:
                    b.copy_(pack_bits(src[:, :mb.size], shape[1] * 8 // self.obs_bits, self.obs_bits))
                else:
                    b[:, :src.shape[1]].copy_(src[:, :b.shape[1]])
                bufs.append(b)
            self.private_obs = True
        else:
            bufs = [obs_buffer, obs_buffer]
            self.private_obs = False
        for b in bufs:
            if b.stride(0) % 16 or b.stride(1) != 1 or b.data_ptr() % 16:
                raise ValueError("obs_buffer must be an int8 (n, pitch) tensor with 16-byte aligned rows")
        self.obs_bufs, self.ld = bufs, bufs[0].stride(0)
        self.obs = bufs[0]
        self.host_block = host_block
        self.readback = list(readback)
        # host_block of shape (vpr, ...): one block per visit of a replay, uploaded
        # with one copy (a 2.5 MB copy runs at ~51 GB/s where 1.25 MB ones reach ~47)
        self.host_per_visit = host_block is not None and self.vpr > 1 and \
            tuple(host_block.shape) == (self.vpr, *bufs[0].shape)
        if host_block is not None:
            if obs_buffer is not None or not host_block.is_pinned() or host_block.dtype != bufs[0].dtype \
                    or not (self.host_per_visit or tuple(host_block.shape) == tuple(bufs[0].shape)) \
                    or not host_block.is_contiguous():
                raise ValueError(f"host_block must be a pinned contiguous {bufs[0].dtype} {tuple(bufs[0].shape)}"
                                 f" (or ({self.vpr}, ...) one block per visit of a replay)")
            for i, b in enumerate(bufs):
                b.copy_(host_block[i % self.vpr] if self.host_per_visit else host_block)
            # uploads run on a copy stream outside the graphs (a copy engine,
            # never SM time), ordered by events against the replays
            self._up_stream = torch.cuda.Stream()
            self._uploaded = [torch.cuda.Event() for _ in bufs]
            self._up_pending = [False] * len(bufs)
            self._read_done = [torch.cuda.Event() for _ in bufs]
            self._read_pending = [False] * len(bufs)
        for dev_t, host_t in self.readback:
            if not host_t.is_pinned() or host_t.numel() * host_t.element_size() < dev_t.numel() * dev_t.element_size():
                raise ValueError("readback targets must be pinned host tensors large enough")
        self._copy_stream = None
        self.upload_done = None  # event of the last host_block upload (see the docstring)
        self._buf_free: list = [None, None]  # event: the last replay reading buffer p has finished
        self.graphs = []
        self._finish_args = []
        self._tev = None
        self.debug_events = None  # a list: per host-fed step, events (upload start, end, replay start, end)
        if timing:
            self._tev = []
            for _ in range(4):
                h = ctypes.c_uint64()
                _lib.call("sg_event_create", ctypes.byref(h))
                self._tev.append(h.value)
        if not eng.tables_fresh:
            raise ValueError("engine tables are stale")
        # keys of the first replayed visit; every replay's finish advances the cursor
        _lib.call("sg_keys_advance", self.table.data_ptr(), self.idx.data_ptr(), kps, self.cur.data_ptr(),
                  stream_handle())
        torch.cuda.synchronize()
        # visit k: count parity k % 2, observation buffer k % len(bufs); graph j holds
        # visits j * vpr ... j * vpr + vpr - 1 of one period lcm(2, len(bufs))
        period = 2 * len(bufs) // math.gcd(2, len(bufs))
        for j in range(period // self.vpr):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for i in range(self.vpr):
                    self._record(j * self.vpr + i)
            self.graphs.append(g)
        torch.cuda.synchronize()

    @staticmethod
    def view_of(mb):
        """The minibatch's device int8 block when the graphs can read it in place
        (16-byte aligned rows), else None (private buffers refilled by step())."""
        v = mb.values
        if isinstance(v, torch.Tensor) and v.is_cuda and v.dtype == torch.int8 and v.stride(1) == 1 \
                and v.stride(0) % 16 == 0 and v.data_ptr() % 16 == 0:
            return v
        return None

    def accepts(self, mb) -> bool:
        """``mb`` can be replayed by these graphs (same minibatch shape, visits left)."""
        return self.replayed < self.planned and mb.size == self.mb.size and int(mb.num_real) == int(self.db.num_real)

    def sweep_ms(self) -> float:
        """Sweep time (ms, all sweeps of the visit) of the last replay (timing=True)."""
        if self._tev is None or not self.replayed:
            raise ValueError("no timed replay")
        p = (self.replayed - 1) % 2
        ms = ctypes.c_float()
        _lib.call("sg_event_elapsed", self._tev[2 * p], self._tev[2 * p + 1], ctypes.byref(ms))
        return float(ms.value)

    @staticmethod
    def obs_geometry(n: int, size: int, obs_bits=8):
        """(shape, dtype) of the private observation buffers (and of a host_block):
        ``obs_bits`` 8 (int8), 4 or 2 (packed rows of a 64-case multiple; True = 4)."""
        bits = 4 if obs_bits is True else (8 if obs_bits is False else int(obs_bits))
        pitch = _pitch(size)
        if bits < 8:
            pitch = max(64, (pitch + 63) // 64 * 64)
            return (n, pitch * bits // 8), torch.uint8
        return (n, pitch), torch.int8

    def _record(self, k: int) -> None:
        eng, db, m, cfg = self.eng, self.db, self.m, self.eng.cfg
        s = stream_handle()
        size = self.mb.size
        cur = self.cur.data_ptr()
        p = k % 2  # count parity
        new, prev = self.cbuf[p], self.cbuf[1 - p]
        obs = self.obs_bufs[k % len(self.obs_bufs)]
        # tables and keys of this visit are ready: the previous replay's finish built/advanced them
        if not eng.use_small:  # the packed sweep checks the block in its own launch
            if self._unpacked is not None:
                u = self._unpacked
                _lib.call("sg_unpack_nibbles" if self.obs_bits == 4 else "sg_unpack_crumbs", obs.data_ptr(),
                          obs.stride(0), u.data_ptr(), u.stride(0), eng.n, size, s)
                _lib.call("sg_check_range", eng.pack.ref, u.data_ptr(), u.stride(0), size, eng.err.ptr, s)
            else:
                _lib.call("sg_check_range", eng.pack.ref, obs.data_ptr(), self.ld, size, eng.err.ptr, s)
        S = cfg.sweeps_per_minibatch
        # step tail: accumulate, CPT update, next tables, clear `prev` (the next
        # replay's count buffer), advance the key cursor
        # the CPT read-back rides in the tail kernel itself (zero-copy store into the pinned tensor)
        cpt_host = next((h for d_, h in self.readback if d_.data_ptr() == eng.cpt.data_ptr()), None)
        tail_check = eng.tail_checks_obs
        f = eng.finish_args(new, prev, 0, key_dev=cur + 8 * S, clear=prev,
                            cursor=(self.table, self.idx, self.kps, self.cur), cpt_host=cpt_host,
                            check=(obs.data_ptr(), self.ld, self.obs_bits, size) if tail_check else None)
        self._finish_args.append(f)
        if self._tev is not None:
            _lib.call("sg_event_record", self._tev[2 * p], s)
        for sw in range(S):
            last = sw == S - 1
            counts_ptr = new.data_ptr() if last else None
            if eng.use_small:
                if sw:
                    eng.sweep_fence(s)
                eng.packed_sweep(db, size, m, 0, cur + 8 * sw, counts_ptr, obs.data_ptr() if last else None, self.ld,
                                 s, obs_bits=self.obs_bits, prefetch_only=tail_check)
            elif eng.rng_mode == _lib.SG_RNG_NUMPY:
                # numpy stream: stream_key(sweep_seed, "var", v) hashed on the device from the
                # cursor's sweep seed (sampler.py:245, rng.py:16-20), then the bit-exact sweep
                site_keys(eng.keys, ":var:", eng.n, seed_dev=cur + 8 * sw)
                eng.numpy_sweep(db, counts_ptr, s)
            else:
                _lib.call("sg_sweep", eng.sweep_net, db.ref, eng.cpt.data_ptr(), eng.ptab.data_ptr(),
                          eng.ftab.data_ptr(), _lib.SG_RNG_FAST, 0, cur + 8 * sw, None, None, None, counts_ptr,
                          eng.err.ptr, s)
        if self._tev is not None:
            _lib.call("sg_event_record", self._tev[2 * p + 1], s)
        if eng.comm is not None:
            eng.comm(new)
        eng.step_tail(f, s)
        for dev_t, host_t in self.readback:  # a kernel node (faster than a D2H memcpy node) into mapped pinned memory
            if host_t is cpt_host:
                continue
            nbytes = dev_t.numel() * dev_t.element_size()
            if nbytes % 8 == 0 and dev_t.data_ptr() % 8 == 0 and host_t.data_ptr() % 8 == 0:
                _lib.call("sg_copy_small", host_t.data_ptr(), dev_t.data_ptr(), nbytes, s)
            else:
                _lib.call("sg_copy_async", host_t.data_ptr(), dev_t.data_ptr(), nbytes, s)

    def step(self, mb=None) -> None:
        """Replay the next planned visit; ``mb`` (optional) refills the observation buffer first."""
        if self.replayed >= self.planned:
            raise IndexError("all planned visits have been replayed")
        p = self.replayed % 2
        main = torch.cuda.current_stream()
        if mb is not None and self.host_block is not None:
            raise ValueError("this graph uploads its own host block; call step() without a minibatch")
        if self.host_block is not None:
            # upload the blocks of the visits two replays ahead (buffers the previous replay
            # read) while this replay runs, so an upload has two replays' time to land
            nb, vpr, k0 = len(self.obs_bufs), self.vpr, self.replayed
            mine = [(k0 + i) % nb for i in range(vpr)]
            gk = (k0 // vpr) % len(self.graphs)
            up = self._up_stream
            dbg = self.debug_events
            if dbg is not None:
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
                ev[0].record(up)
            if self.host_per_visit:  # the replay's vpr consecutive buffers in one copy
                qs = [(k0 + 2 * vpr + i) % nb for i in range(vpr)]
                for q in qs:
                    if self._read_pending[q]:
                        up.wait_event(self._read_done[q])
                first = self.obs_bufs[qs[0]]
                _lib.call("sg_copy_async", first.data_ptr(), self.host_block.data_ptr(),
                          vpr * first.numel() * first.element_size(), up.cuda_stream)
                for q in qs:
                    self._uploaded[q].record(up)
                    self.upload_done = self._uploaded[q]
                    self._up_pending[q] = True
            for i in range(0 if self.host_per_visit else vpr):
                q = (k0 + 2 * vpr + i) % nb
                if self._read_pending[q]:
                    up.wait_event(self._read_done[q])  # the replay that last read buffer q has finished
                nxt = self.obs_bufs[q]
                _lib.call("sg_copy_async", nxt.data_ptr(), self.host_block.data_ptr(),
                          nxt.numel() * nxt.element_size(), up.cuda_stream)
                self._uploaded[q].record(up)
                self.upload_done = self._uploaded[q]
                self._up_pending[q] = True
            if dbg is not None:
                ev[1].record(up)
            for p in mine:
                if self._up_pending[p]:
                    main.wait_event(self._uploaded[p])
                    self._up_pending[p] = False
            if dbg is not None:
                ev[2].record(main)
            self.graphs[gk].replay()
            if dbg is not None:
                ev[3].record(main)
                dbg.append(ev)
            for p in mine:
                self._read_done[p].record(main)
                self._read_pending[p] = True
            self.replayed += vpr
            _lib.launch_count += self.launches_per_step * vpr
            return
        if self.vpr > 1:
            if mb is not None:
                raise ValueError("two visits per replay take no minibatch")
            self.graphs[(self.replayed // 2) % len(self.graphs)].replay()
            self.replayed += 2
            _lib.launch_count += self.launches_per_step * 2
            return
        if mb is not None:
            vals = mb.values
            buf = self.obs_bufs[p]
            if not (isinstance(vals, torch.Tensor) and vals.is_cuda and vals.data_ptr() == buf.data_ptr()):
                if isinstance(vals, torch.Tensor) and vals.is_cuda:
                    src = vals
                else:  # host block: range-checked before the int8 conversion (as _obs_for does)
                    host = vals.numpy() if isinstance(vals, torch.Tensor) else np.asarray(vals)
                    if not self.nibbles:
                        cards = np.asarray(self.eng.net.cardinalities)[:, None]
                        if ((host >= cards) | (host < -1)).any():
                            raise ValidationError("data contains a state >= its variable's cardinality")
                    src = torch.from_numpy(np.ascontiguousarray(host.astype(np.uint8 if self.nibbles else np.int8)))
                if self.nibbles and (src.dtype != torch.uint8 or tuple(src.shape) != tuple(buf.shape)):
                    raise ValueError(f"expected a packed block uint8 {tuple(buf.shape)} (io.pack_bits)")
                if not self.private_obs or src.is_cuda:
                    # device blocks are produced on this stream: copy in stream order
                    if self.nibbles:
                        buf.copy_(src, non_blocking=True)
                    else:
                        copy_rows(buf, src, mb.size)
                else:
                    # upload on the copy stream once the replay that last read this buffer is done,
                    # so it overlaps the other parity's replay
                    if self._copy_stream is None:
                        self._copy_stream = torch.cuda.Stream()
                    cs = self._copy_stream
                    if self._buf_free[p] is not None:
                        cs.wait_event(self._buf_free[p])
                    with torch.cuda.stream(cs):
                        if self.nibbles:
                            buf.copy_(src, non_blocking=True)
                        else:
                            buf[:, :mb.size].copy_(src, non_blocking=True)
                    main.wait_stream(cs)
        self.graphs[p].replay()
        if self.private_obs:
            ev = torch.cuda.Event()
            ev.record(main)
            self._buf_free[p] = ev
        self.replayed += 1
        _lib.launch_count += self.launches_per_step

    @property
    def launches_per_step(self) -> int:
        eng = self.eng
        one_cta = eng.pack.cells <= 4096  # sg_step_finish is one kernel, else six launches
        # the CPTs' read-back is stored by the tail kernel (one copy launch inside the multi-launch tail)
        cpt_rb = any(d_.data_ptr() == eng.cpt.data_ptr() for d_, _ in self.readback)
        readback = len(self.readback) - (1 if cpt_rb and one_cta else 0)
        # the packed sweep folds in the range check; a packed block on the generic path is unpacked first
        check = 0 if eng.use_small else (2 if self._unpacked is not None else 1)
        keys = eng.cfg.sweeps_per_minibatch if eng.rng_mode == _lib.SG_RNG_NUMPY else 0
        if eng.use_small:
            keys += eng.cfg.sweeps_per_minibatch - 1  # sweep fences
        return (check + keys + eng.cfg.sweeps_per_minibatch + (1 if one_cta else 5 + (1 if eng.use_small else 0))
                + readback)

    def finish(self) -> None:
        """Hand the last visit's counts back to the engine's moving-sum bookkeeping."""
        if self.replayed:
            self.eng.prev_counts[self.mb.index] = self.cbuf[(self.replayed - 1) % 2].clone()


class StreamGraphs:
    """CUDA-graph replay of FRESH minibatch visits: the out-of-core mode of the
    packed and joint paths (exponential accumulator, sampler.py:346-351 and
    :434-441 -- every visit re-initialises its latents).

    One replay = [decode of a packed .sgb block] + ``sg_small_prepare`` (cases
    bucketed by latent pattern, observed fields from the block, FAST initial
    latents keyed derive_seed(seed, "latent_init", pass, mb) read from the
    key cursor) + the sweep(s) + the step tail.  The block is the graph's
    private buffer (two, alternating), refilled by :meth:`step` from each
    streamed minibatch, so every replay samples the minibatch it was given.
    ``visits``: the planned (pass, minibatch) sequence of full minibatches;
    replays equal eager visits bit for bit."""

    def __init__(self, eng: Engine, size: int, m: int, visits, obs_bits: int = 8, readback=()):
        cfg = eng.cfg
        if cfg.accumulator_mode != "exponential" or not eng.use_small:
            raise ValueError("stream graphs replay fresh visits of the packed / joint path (exponential accumulator)")
        if obs_bits not in (8, 4, 2):
            raise ValueError("obs_bits must be 8, 4 or 2")
        if obs_bits < 8 and not eng.joint:
            raise ValueError("packed observation blocks are range-checked by the joint sweep only")
        if not eng.tables_fresh:
            raise ValueError("engine tables are stale: run one eager visit first")
        self.eng, self.size, self.m = eng, size, m
        self.obs_bits = int(obs_bits)
        S = cfg.sweeps_per_minibatch
        self.kps = kps = S + 2  # sweep keys, Dirichlet key, latent-init key
        visits = list(visits)
        table = np.empty((len(visits), kps), dtype=np.uint64)
        for i, (p, b) in enumerate(visits):
            for sw in range(S):
                table[i, sw] = derive_seed(cfg.seed, "sweep", p, b, sw)
            table[i, S] = derive_seed(derive_seed(cfg.seed, "cpt_update", p, b), "sample_cpts")
            table[i, S + 1] = derive_seed(cfg.seed, "latent_init", p, b)
        d = eng.dev
        self.visits = visits
        self.table = torch.from_numpy(table.view(np.int64)).to(d)
        self.idx = torch.zeros(1, dtype=torch.int32, device=d)
        self.cur = torch.zeros(kps, dtype=torch.int64, device=d)
        self.planned, self.replayed = len(visits), 0
        self.db = SmallBatch(eng.n, m, size, d)
        self.db.num_real = size
        self.cbuf = [torch.zeros_like(eng.counts), torch.zeros_like(eng.counts)]
        shape, dt = StepGraphs.obs_geometry(eng.n, size, self.obs_bits)
        self.obs_bufs = [torch.full(shape, -1 if dt == torch.int8 else 0xFF, dtype=dt, device=d) for _ in range(2)]
        self.ld = self.obs_bufs[0].stride(0)
        self._int8 = None
        if self.obs_bits < 8:  # the prepare step reads int8 rows
            self._int8 = torch.empty((eng.n, _pitch(size)), dtype=torch.int8, device=d)
        self.readback = list(readback)
        self._buf_free = [None, None]
        self._copy_stream = None
        _lib.call("sg_keys_advance", self.table.data_ptr(), self.idx.data_ptr(), kps, self.cur.data_ptr(),
                  stream_handle())
        torch.cuda.synchronize()
        self.graphs = []
        for parity in (0, 1):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._record(parity)
            self.graphs.append(g)
        torch.cuda.synchronize()

    def _record(self, p: int) -> None:
        eng, db, m, S = self.eng, self.db, self.m, self.eng.cfg.sweeps_per_minibatch
        s = stream_handle()
        cur = self.cur.data_ptr()
        obs = self.obs_bufs[p]
        prep, prep_ld = obs, self.ld
        if self._int8 is not None:
            u = self._int8
            _lib.call("sg_unpack_nibbles" if self.obs_bits == 4 else "sg_unpack_crumbs", obs.data_ptr(), obs.stride(0),
                      u.data_ptr(), u.stride(0), eng.n, self.size, s)
            prep, prep_ld = u, u.stride(0)
        _lib.call("sg_small_prepare", eng.pack.small_ref, prep.data_ptr(), prep_ld, self.size, m, eng.case_base, 0, 1,
                  db.scratch.data_ptr(), db.pattern.data_ptr(), db.case_id.data_ptr(), db.lanes.data_ptr(), db.lane_ld,
                  cur + 8 * (S + 1), s)
        new = self.cbuf[p]
        cpt_host = next((h for d_, h in self.readback if d_.data_ptr() == eng.cpt.data_ptr()), None)
        tail_check = eng.tail_checks_obs
        f = eng.finish_args(new, None, 0, key_dev=cur + 8 * S, clear=self.cbuf[1 - p],
                            cursor=(self.table, self.idx, self.kps, self.cur), cpt_host=cpt_host,
                            check=(obs.data_ptr(), self.ld, self.obs_bits, self.size) if tail_check else None)
        self._f = getattr(self, "_f", []) + [f]
        for sw in range(S):
            last = sw == S - 1
            if sw:
                eng.sweep_fence(s)
            eng.packed_sweep(db, self.size, m, 0, cur + 8 * sw, new.data_ptr() if last else None,
                             obs.data_ptr() if last else None, self.ld, s, obs_bits=self.obs_bits,
                             prefetch_only=tail_check)
        if eng.comm is not None:
            eng.comm(new)
        eng.step_tail(f, s)
        for dev_t, host_t in self.readback:
            if host_t is not cpt_host:  # the CPTs are stored by the tail kernel itself
                _lib.call("sg_copy_small", host_t.data_ptr(), dev_t.data_ptr(), dev_t.numel() * dev_t.element_size(), s)

    def step(self, mb) -> None:
        """Replay the next planned visit on minibatch ``mb`` (its block is copied into the graph's buffer:
        device blocks in stream order, host blocks on a copy stream after the buffer's last reader)."""
        if self.replayed >= self.planned:
            raise IndexError("all planned visits have been replayed")
        if mb.size != self.size or int(mb.num_real) != self.size:
            raise ValueError("stream graphs replay full minibatches of the captured size")
        p = self.replayed % 2
        buf = self.obs_bufs[p]
        vals = mb.values
        main = torch.cuda.current_stream()
        if isinstance(vals, torch.Tensor) and vals.is_cuda:
            if self.obs_bits < 8 and (vals.dtype != torch.uint8 or tuple(vals.shape) != tuple(buf.shape)):
                from .io import pack_bits

                vals = pack_bits(vals, buf.shape[1] * 8 // self.obs_bits, self.obs_bits)
            if self.obs_bits < 8:
                buf.copy_(vals, non_blocking=True)
            else:
                copy_rows(buf, vals, self.size)
        else:
            host = vals.numpy() if isinstance(vals, torch.Tensor) else np.asarray(vals)
            if self.obs_bits == 8:
                cards = np.asarray(self.eng.net.cardinalities)[:, None]
                if ((host >= cards) | (host < -1)).any():
                    raise ValidationError("data contains a state >= its variable's cardinality")
            src = torch.from_numpy(np.ascontiguousarray(host.astype(np.uint8 if self.obs_bits < 8 else np.int8)))
            if self._copy_stream is None:
                self._copy_stream = torch.cuda.Stream()
            cs = self._copy_stream
            if self._buf_free[p] is not None:
                cs.wait_event(self._buf_free[p])
            with torch.cuda.stream(cs):
                if self.obs_bits < 8:
                    buf.copy_(src, non_blocking=True)
                else:
                    buf[:, :self.size].copy_(src, non_blocking=True)
            main.wait_stream(cs)
        self.graphs[p].replay()
        ev = torch.cuda.Event()
        ev.record(main)
        self._buf_free[p] = ev
        self.replayed += 1
        _lib.launch_count += self.launches_per_step

    @property
    def launches_per_step(self) -> int:
        S = self.eng.cfg.sweeps_per_minibatch
        cpt_rb = any(d_.data_ptr() == self.eng.cpt.data_ptr() for d_, _ in self.readback)
        return (1 if self._int8 is not None else 0) + 3 + (S - 1) + S + 1 + len(self.readback) - (1 if cpt_rb else 0)

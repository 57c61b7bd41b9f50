#!/usr/bin/env python
"""Benchmark of the SAME Gibbs hot path (BASELINE.json metric: node-samples/s).

Default workload (BASELINE.json configs[1], "C2"): Koller student network, 1M
cases per GPU, 50% of cells hidden, SAME m = 10, one minibatch of 1M cases,
moving-sum accumulator, sampled Dirichlet CPT update, fast RNG mode.  One step
= one minibatch visit = sweep/tally + accumulator + Dirichlet update + next
conditional tables (+ the count all-reduce when N > 1).  Synthetic data of
that shape comes from the reference's own forward_sample/mask streams,
generated on the device.  node-samples per step = n_vars x cases x m
(sampler.py:475).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload c2|c3|c4|c5]

``--workload c3`` (MOOC-shaped, 334 variables, 131,010 cases, m = 5) and
``c4`` (random DAG, 1000 nodes, 1.25M cases per GPU = 10M over 8, m = 1, 30%
missing) measure the generic kernel on the other BASELINE shapes; ``c5``
streams a 10^7-case 4-bit .sgb file of the 1000-node network per GPU
(BinaryFileSource: disk -> pinned -> device one block ahead), m = 20,
exponential accumulator, one full pass timed.
C2 is the headline line.

Timing: per-step CUDA events on the launching stream, L2 flushed (256 MB
write + 256 MB read) between timed steps, max over ranks.  Prints ONE JSON
line on rank 0.  ``--impl reference`` times the CPU oracle (NumPy restatement
of the reference, oracle/) on the host cores instead.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "node-samples/sec"
UNIT = "node-samples/s"


class Workload:
    """One BASELINE configuration: network, data shape, SAME factor."""

    def __init__(self, key, title, cases, m, latent, cpu_cases):
        self.key, self.title, self.cases, self.m = key, title, cases, m
        self.latent = latent          # latent fraction f of the cells
        self.cpu_cases = cpu_cases    # case slice of one CPU oracle process

    # -- network + generating CPTs (package types)
    def network(self):
        if self.key == "c2":
            from paper_1511_06416_b200.io import bundled_network_path, load_network_file

            return load_network_file(bundled_network_path("koller"))
        from paper_1511_06416_b200 import netgen

        if self.key == "c3":
            net = netgen.mooc_network(15, 319, seed=3)
            return net, netgen.dirichlet_cpts(net, 1.0, seed=6)
        net = netgen.random_dag_network(1000, max_parents=4, min_card=2, max_card=4, seed=4)
        return net, netgen.dirichlet_cpts(net, 1.0, seed=5)  # C4 and C5 share the network

    # -- device observations of this rank's shard
    def observations(self, net, truth, rank):
        import paper_1511_06416_b200 as sg
        from paper_1511_06416_b200 import netgen

        base = rank * self.cases
        if self.key == "c3":
            return netgen.mooc_observations(net, truth, self.cases, 15, density=0.022, seed=103, case_base=base)
        hide, seed = (0.5, 100) if self.key == "c2" else (0.3, 104)
        return sg.forward_sample_device(net, truth, self.cases, seed=seed, hide_fraction=hide, mask_seed=seed + 100,
                                        case_base=base)

    # -- CPU oracle of the same shape (dense int32, -1 = missing)
    def oracle_problem(self, cases, slice_id):
        import numpy as np

        import oracle as O

        if self.key == "c2":
            net, truth = O.koller()
            dense = O.mask_dense(O.forward_sample(net, truth, cases, 100 + slice_id), 0.5, 200 + slice_id)
            return net, dense
        pnet, ptruth = self.network()
        net = O.make_net(list(pnet.cardinalities),
                         [(p, c) for c in range(pnet.num_vars) for p in pnet.parents[c]])
        dense = O.forward_sample(net, ptruth.tables, cases, 100 + slice_id)
        rng = np.random.default_rng(200 + slice_id)
        if self.key == "c3":
            dense = np.where(rng.random(dense.shape) < 0.022, dense, -1).astype(np.int32)
            dense[:15] = -1
        else:
            dense = np.where(rng.random(dense.shape) < 0.3, -1, dense).astype(np.int32)
        return net, dense

    def config(self, n_gpus: int, rng: str, n_vars: int) -> dict:
        return {
            "workload": self.title, "network": {"c2": "koller-student", "c3": "mooc-shaped",
                                                "c4": "random-dag-1000", "c5": "random-dag-1000"}[self.key],
            "n_vars": n_vars, "cases_per_gpu": self.cases, "global_minibatch": self.cases * n_gpus, "m": self.m,
            "latent_fraction": round(self.latent, 4), "rng": rng,
            "parallelism": f"case-sharded x{n_gpus}, int64 count all-reduce" if n_gpus > 1 else "single GPU",
            "l2": "flushed between timed steps (sg_flush_l2: 256 MB write + 256 MB read, outside the step events)",
        }


WORKLOADS = {
    "c2": Workload("c2", "C2: koller-student (5 vars), 1M cases/GPU, 50% hidden, SAME m=10, minibatch=1M, "
                         "moving-sum, Dirichlet CPT update", 1_000_000, 10, 0.5, 100_000),
    "c3": Workload("c3", "C3: MOOC-shaped (15 latent concepts + 319 questions), 131,010 cases, 2.2% of responses "
                         "observed, SAME m=5, minibatch=all, moving-sum, Dirichlet CPT update", 131_010, 5, 0.978,
                   8_000),
    "c4": Workload("c4", "C4: random DAG, 1000 nodes, in-degree<=4, cards 2-4, 1.25M cases/GPU (10M over 8), "
                         "30% missing, SAME m=1, minibatch=shard, moving-sum, Dirichlet CPT update", 1_250_000, 1,
                   0.3, 4_000),
    "c5": Workload("c5", "C5: out-of-core, random DAG 1000 nodes, 30% missing, SAME m=20, one pass over a 4-bit "
                         ".sgb file of 10^7 cases per GPU (minibatches of 131,072 cases, disk -> pinned -> device), "
                         "exponential accumulator, Dirichlet CPT update", 131_072, 20, 0.3, 500),
}


# ---------------------------------------------------------------- CPU oracle legs

def _oracle_worker(args):
    """Time oracle steps (sweep + tally + moving sum + Dirichlet) on a case slice."""
    key, cases, steps, budget_s, slice_id = args
    import numpy as np

    import oracle as O

    wl = WORKLOADS[key]
    net, dense = wl.oracle_problem(cases, slice_id)
    groups = O.greedy_coloring(net)
    cur = O.init_cpts(net, 300)
    total = [np.zeros((net.rows(v), net.cards[v])) for v in range(net.n)]
    values, missing = O.replicate(dense, wl.m)
    weights = np.ones(values.shape[1])
    O.init_latent(net, values, missing, 300, 0, 0)
    prev = None
    times = []
    t_start = time.perf_counter()
    for s in range(steps):
        t0 = time.perf_counter()
        counts = O.sweep(net, groups, cur, values, missing, weights, O.site_seed(300, "sweep", s, 0, 0))
        O.moving_sum(total, prev, counts)
        prev = counts
        cur = O.sample_cpts(total, [1.0] * net.n, O.site_seed(300, "cpt_update", s, 0))
        times.append(time.perf_counter() - t0)
        if budget_s and time.perf_counter() - t_start > budget_s:
            break
    return times


REF_DIR = ROOT / "oracle" / "_ref"  # the unmodified reference, installed by oracle/build_ref.sh


def have_reference() -> bool:
    return (REF_DIR / "samegibbs" / "__init__.py").exists()


def _reference_worker(args):
    """Time the UNMODIFIED reference's own ``samegibbs.run(threads=1)`` (oracle/_ref)
    on a case slice of the workload: one pass = one minibatch visit (sweep +
    tally + accumulator + Dirichlet update); per-pass times from its trace."""
    key, cases, passes, slice_id = args
    sys.path.insert(0, str(REF_DIR))
    import samegibbs as R

    wl = WORKLOADS[key]
    onet, dense = wl.oracle_problem(cases, slice_id)  # the same data the port times (bit-exact generators)
    net = R.build_network(list(onet.cards), [(p, c) for c in range(onet.n) for p in onet.parents[c]])
    data = R.DataMatrix.from_dense(dense)
    mode = "exponential" if key == "c5" else "moving_sum"
    cfg = R.SamplerConfig(same_m=wl.m, minibatch_size=cases, num_passes=passes, seed=300, accumulator_mode=mode,
                          exp_decay=0.9 if mode == "exponential" else 1.0)
    _, trace = R.run(net, data, cfg, threads=1)
    secs = [r.seconds for r in trace.records]
    return [b - a for a, b in zip([0.0] + secs[:-1], secs)]


def _cpu_times(key, cases, steps, slice_id):
    if have_reference():
        return _reference_worker((key, cases, steps, slice_id)), "reference"
    return _oracle_worker((key, cases, steps, 0, slice_id)), "port"


def cpu_baseline(wl: Workload, n_vars: int, budget_s: float = 12.0) -> dict:
    """Single core, rank 0, N=1: the reference's own run() (oracle/_ref) on a case
    slice of the workload, else the oracle port."""
    cases = wl.cpu_cases
    # about budget_s of CPU time at ~1e7 node-samples/s
    passes = int(max(4, min(40, budget_s * 1e7 / (n_vars * cases * wl.m))))
    times, kind = _cpu_times(wl.key, cases, passes, 0)
    per = statistics.median(times[1:] if len(times) > 2 else times)
    what = ("samegibbs.run(threads=1) of the unmodified reference (oracle/_ref)" if kind == "reference" else
            "oracle (NumPy restatement of samegibbs), sweep+tally+moving-sum+Dirichlet per step")
    return {"value": n_vars * cases * wl.m / per, "unit": UNIT, "cores": 1, "kind": kind,
            "sample": f"{what}, single process, {cases}-case slice x m={wl.m}, {len(times)} passes of one "
                      f"minibatch, median pass {per * 1e3:.1f} ms"}


def _arm_worker(args):
    key, cases, steps, slice_id = args
    return _cpu_times(key, cases, steps, slice_id)[0]


def reference_arm(args, wl: Workload) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import multiprocessing as mp

    n_vars = wl.network()[0].num_vars
    procs = max(1, min(os.cpu_count() or 1, 64))
    total_steps = args.steps + args.warmup
    # bound the run to roughly a minute of CPU time per process (~1e7 node-samples/s per core)
    cases = int(min(wl.cpu_cases, max(1_000, 60.0 / total_steps * 1e7 / (n_vars * wl.m))) // 500 * 500)
    cases = max(cases, 500)
    kind = "reference" if have_reference() else "port"
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(procs) as pool:
        res = pool.map(_arm_worker, [(wl.key, cases, total_steps, i) for i in range(procs)])
    wall = time.perf_counter() - t0
    timed = [r[args.warmup:] for r in res]
    per_step = max(sum(t) for t in timed) / max(1, args.steps)  # slowest worker bounds the aggregate
    value = procs * n_vars * cases * wl.m / per_step
    what = ("the unmodified reference's samegibbs.run(threads=1) (oracle/_ref, built by oracle/build_ref.sh)"
            if kind == "reference" else "the oracle port (NumPy restatement)")
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": wl.config(args.gpus, "numpy", n_vars),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": kind,
                         "sample": f"{procs} independent single-threaded processes of {what}, each on its own "
                                   f"{cases}-case slice x m={wl.m}, one minibatch visit per step (aggregate upper "
                                   f"bound; the reference's own threads knob does not scale), wall {wall:.1f} s"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))


# ---------------------------------------------------------------- clocks

class ClockSampler:
    """NVML samples of SM clock and throttle reasons during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001 - clocks are best effort metadata
            self.nvml = None

    def _loop(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nvml.nvmlDeviceGetClockInfo(self.h, self.nvml.NVML_CLOCK_SM))
                mask = self.nvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nvml:
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.nvml:
            self.t.join()

    def summary(self) -> dict:
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------- our arm

def load_traffic(wl: Workload, kernel: str):
    """Per-launch DRAM bytes of the sweep kernel from the committed ncu summary (or None)."""
    for p in sorted((ROOT / "profiles").glob("ncu_sweep_*.json"), reverse=True):
        try:
            d = json.loads(p.read_text())
            base = d.get("kernel", "").split(" ")[0].split("<")[0]
            if (d.get("workload", "c2") == wl.key and base == kernel.split(" ")[0]
                    and d.get("cases") == wl.cases and d.get("m") == wl.m):
                return d.get("dram_bytes_per_launch"), p.name
        except Exception:  # noqa: BLE001
            continue
    return None, None


def event_floor_ms(eng, flush_l2) -> float | None:
    """Events-around-an-empty-kernel time (the sweep's launch shape, in a graph)."""
    import ctypes

    import torch

    from paper_1511_06416_b200 import _lib

    if not getattr(eng, "joint", False):
        return None
    ev = []
    for _ in range(2):
        h = ctypes.c_uint64()
        _lib.call("sg_event_create", ctypes.byref(h))
        ev.append(h.value)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        s = torch.cuda.current_stream().cuda_stream
        _lib.call("sg_event_record", ev[0], s)
        _lib.call("sg_noop", sms - 1, 1024, 120 * 1024, s)
        _lib.call("sg_event_record", ev[1], s)
    out = []
    for k in range(15):
        flush_l2(k)
        g.replay()
        torch.cuda.synchronize()
        ms = ctypes.c_float()
        _lib.call("sg_event_elapsed", ev[0], ev[1], ctypes.byref(ms))
        if k >= 3:
            out.append(ms.value)
    for h in ev:
        _lib.call("sg_event_destroy", h)
    return statistics.mean(out)


def our_arm(args, wl: Workload) -> None:
    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_1511_06416_b200 as sg
    from paper_1511_06416_b200 import _lib
    from paper_1511_06416_b200.engine import Engine, StepGraphs

    CASES, M = wl.cases, wl.m
    net, truth = wl.network()
    n_vars = net.num_vars
    if args.rng == "auto":
        from paper_1511_06416_b200.device import netpack

        args.rng = "joint" if netpack(net).joint is not None and M <= 32 else "fast"
    cfg = sg.SamplerConfig(same_m=M, minibatch_size=CASES, num_passes=1, seed=300, rng=args.rng)
    obs = wl.observations(net, truth, rank)
    comm = (lambda c: dist.all_reduce(c)) if world > 1 else None
    eng = Engine(net, cfg, case_base=rank * CASES, comm=comm)
    mb = next(iter(sg.DeviceSource(obs, CASES, CASES)))
    latent = float((obs[:, :CASES] < 0).float().mean())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    flush_rd = torch.ones(32 << 20, dtype=torch.int64, device="cuda")  # 256 MB

    def flush_l2(k):
        # evict the working set: write 256 MB (> 126 MB L2), then read another
        # 256 MB so the flush's own dirty lines are written back here, outside
        # the timed events, not during the next step.  sg_flush_l2's kernels
        # prefer the sweep's max-shared carveout, so the timed step does not
        # start with an L1/shared reconfiguration that back-to-back steps never see
        _lib.call("sg_flush_l2", flush.data_ptr(), flush_rd.data_ptr(), 256 << 20, k & 0xFFFFFFFF,
                  torch.cuda.current_stream().cuda_stream)

    # eager warm-up visits: the first one builds the resident lanes
    for w in range(args.warmup):
        eng.visit(mb, w, M)
    torch.cuda.synchronize()
    e2e_steps = max(4, min(args.steps, 200)) // 2 * 2  # long enough that one host hiccup does not dominate
    graph_warm = 3
    first = args.warmup
    graphs = None
    if not args.eager:
        total_replays = graph_warm + args.steps + 2 + e2e_steps
        # private double-buffered observation blocks: e2e steps upload the next block
        # on a copy stream while the current visit runs
        # joint path: observation blocks travel in the 4-bit .sgb form (half the PCIe bytes)
        obs_bits = 8
        # the observation block travels packed: 2 bits/cell when every card <= 3, else 4
        # (joint sweep: read packed; generic sweep: unpacked + range-checked in the graph)
        if (eng.joint or not eng.use_small) and max(net.cardinalities) <= 15:
            obs_bits = 2 if max(net.cardinalities) <= 3 else 4
        graphs = StepGraphs(eng, mb, M, range(first, first + total_replays), obs_bits=obs_bits)
        for _ in range(graph_warm):
            graphs.step()
        first += graph_warm
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
        torch.cuda.synchronize()

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches0 = _lib.launch_count
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush_l2(k)
            starts[k].record()
            if graphs is not None:
                graphs.step()
            else:
                eng.visit(mb, first + k, M)
            ends[k].record()
        torch.cuda.synchronize()
    launches = _lib.launch_count - launches0
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    err = eng.err.read()
    if err:
        raise RuntimeError(f"device error word {err}")
    ms = statistics.mean(step_ms)
    # the sweep kernel alone, L2 flushed before every step: with graph replay, external timing
    # events recorded inside the step graph around the sweep node (the kernel as it runs in
    # the replayed step); eager mode: events around its launch in eager visits
    t_first = first + args.steps + 40 + e2e_steps
    if graphs is not None:
        graphs.finish()
        tg = StepGraphs(eng, mb, M, range(t_first, t_first + 25), obs_bits=graphs.obs_bits, timing=True)
        sweep_ms = []
        for k in range(25):
            flush_l2(k)
            tg.step()
            torch.cuda.synchronize()
            if k >= 3:
                sweep_ms.append(tg.sweep_ms() / cfg.sweeps_per_minibatch)
        tg.finish()
        graphs.finish = lambda: None  # the engine's moving-sum state already holds the timing visits
        # timing floor of this method: an EMPTY kernel of the sweep's launch shape, bracketed by
        # the same external events inside a captured graph, L2 flushed before each replay
        floor_ms = event_floor_ms(eng, flush_l2)
    else:
        eng.sweep_events = []
        for k in range(20):
            flush_l2(k)
            # keep the device busy (a spin kernel, no memory traffic) while the host enqueues the
            # visit, so the events around the sweep time the kernel, not the host's launch latency
            torch.cuda._sleep(200_000)
            eng.visit(mb, t_first + k, M)
        torch.cuda.synchronize()
        sweep_ms = [a.elapsed_time(b) / nsw for a, b, nsw in eng.sweep_events[2:]]
        eng.sweep_events = None
        floor_ms = None
    sw = statistics.mean(sweep_ms)
    if world > 1:
        t = torch.tensor([ms, sw], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, sw = float(t[0]), float(t[1])
    node_samples = n_vars * CASES * M  # per GPU per step
    value = world * node_samples / (ms * 1e-3)

    # ---- e2e through the public API: pinned host minibatch -> device, step, CPTs back to host
    if graphs is not None and graphs.nibbles:
        from paper_1511_06416_b200.io import pack_bits

        shape, _ = StepGraphs.obs_geometry(n_vars, CASES, graphs.obs_bits)
        host_obs = torch.empty(shape, dtype=torch.uint8, pin_memory=True)
        # the minibatch as a packed .sgb block
        host_obs.copy_(pack_bits(obs[:, :CASES], shape[1] * 8 // graphs.obs_bits, graphs.obs_bits).cpu())
    elif graphs is not None:  # int8 block in the graphs' buffer layout (missing-padded to the row pitch)
        shape, _ = StepGraphs.obs_geometry(n_vars, CASES)
        host_obs = torch.full(shape, -1, dtype=torch.int8).pin_memory()
        host_obs[:, :CASES].copy_(obs[:, :CASES])
    else:
        host_obs = torch.empty((n_vars, CASES), dtype=torch.int8, pin_memory=True)
        host_obs.copy_(obs[:, :CASES])
    hmb = sg.Minibatch(index=0, values=host_obs, weights=np.ones(CASES), num_real=CASES)
    cpt_host = torch.empty(eng.pack.cells, dtype=torch.float64, pin_memory=True)
    e2e_graphs = None
    if graphs is not None:
        # host-fed step graphs: each step() uploads the pinned blocks of the visits two
        # ahead on a copy stream overlapped with the replay; every visit's tail stores its
        # CPTs into pinned host memory; two visits per graph replay
        graphs.finish()
        # one pinned block per visit of a replay (the same minibatch twice): a
        # replay's two uploads go as one copy
        host_visits = torch.empty((2, *host_obs.shape), dtype=host_obs.dtype, pin_memory=True)
        host_visits.copy_(host_obs.expand(2, *host_obs.shape))
        e2e_graphs = StepGraphs(eng, mb, M, range(first + args.steps + 10, first + args.steps + 20 + e2e_steps),
                                obs_bits=graphs.obs_bits, host_block=host_visits, readback=[(eng.cpt, cpt_host)],
                                visits_per_replay=2)
    per_call = e2e_graphs.vpr if e2e_graphs is not None else 1  # visits per e2e_step() call
    e2e_calls = e2e_steps // per_call

    ready = [torch.cuda.Event(), torch.cuda.Event()]

    def e2e_step(k):
        if e2e_graphs is not None:
            e2e_graphs.step()  # H2D of the next block (copy stream) || replay: sweep -> tail -> CPTs to host
        else:
            eng.visit(hmb, 20_000 + k, M)
            cpt_host.copy_(eng.cpt, non_blocking=True)
        ready[k % 2].record()  # the host may read this step's CPTs once it has completed

    # The PCIe link drops to a low-power state while the device-only steps run;
    # bring it back to full speed before the e2e region, as a streaming
    # pipeline would keep it: upload blocks until three consecutive rounds
    # reach >= 85 % of the best H2D rate seen, for at least 250 ms (measured on
    # the B200 boxes: after device-only work the H2D rate can sit at 2-15 GB/s
    # for 50-100 ms before it returns to ~47 GB/s), and while the best rate is
    # below 30 GB/s for up to 2 s.
    scratch = torch.empty_like(host_obs, device="cuda")
    t_warm = time.perf_counter()
    best, good, rates = 0.0, 0, []
    ew0, ew1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    while True:
        ew0.record()
        for _ in range(8):
            scratch.copy_(host_obs, non_blocking=True)
        ew1.record()
        torch.cuda.synchronize()
        rate = 8 * host_obs.numel() * host_obs.element_size() / (ew0.elapsed_time(ew1) * 1e-3) / 1e9
        rates.append(rate)
        best = max(best, rate)
        good = good + 1 if rate >= 0.85 * best else 0
        el = time.perf_counter() - t_warm
        if (el >= 0.25 and good >= 3 and best >= 30.0) or el >= 2.0:
            break
    h2d_warm = {"gbs_last": round(rates[-1], 1), "gbs_best": round(best, 1), "rounds": len(rates),
                "ms": round((time.perf_counter() - t_warm) * 1e3, 1)}
    del scratch
    for w in range(2):
        e2e_step(w)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dbg = [torch.cuda.Event(enable_timing=True) for _ in range(e2e_calls)] if os.environ.get("SG_E2E_DEBUG") else None
    if dbg and e2e_graphs is not None:
        e2e_graphs.debug_events = []
    with ClockSampler(local) as e2e_clk:
        e0.record()
        h0 = time.perf_counter()
        for k in range(e2e_calls):
            e2e_step(k)
            if dbg:
                dbg[k].record()
        e1.record()
        host_enqueue_us = (time.perf_counter() - h0) * 1e6 / e2e_steps
        torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / e2e_steps
    if dbg:
        print("e2e per-call us:", [round((dbg[k].elapsed_time(dbg[k + 1])) * 1e3, 1) for k in range(e2e_calls - 1)],
              file=sys.stderr)
        if e2e_graphs is not None and e2e_graphs.debug_events:
            for k, ev in enumerate(e2e_graphs.debug_events[10:16]):
                print(f"step {k + 10}: upload {e0.elapsed_time(ev[0]) * 1e3:8.1f} -> {e0.elapsed_time(ev[1]) * 1e3:8.1f}"
                      f"  replay {e0.elapsed_time(ev[2]) * 1e3:8.1f} -> {e0.elapsed_time(ev[3]) * 1e3:8.1f} us",
                      file=sys.stderr)
        print("e2e clocks:", e2e_clk.summary(), "host enqueue us/step:", round(host_enqueue_us, 1), file=sys.stderr)
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t[0])
    e2e_value = world * node_samples / (e2e_ms * 1e-3)

    if rank == 0:
        try:
            peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
            peak, peak_src = float(peaks["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy)"
        except Exception:  # noqa: BLE001
            peak, peak_src = 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"
        bpns = 1.0 + latent
        algo_bytes = bpns * node_samples
        achieved = algo_bytes / (sw * 1e-3) / 1e9
        kernel = ("k_joint_sweep (sg_joint_sweep)" if eng.joint else
                  "k_small_sweep (sg_small_sweep)" if eng.use_small else "k_sweep (sg_sweep)")
        traffic, traffic_src = load_traffic(wl, kernel)
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int8 states, u32 draws, f64 CPTs", "data": "synthetic",
            "config": wl.config(world, args.rng, n_vars),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "kernel": kernel,
                         "kernel_ms": sw, "algorithmic_bytes_per_launch": algo_bytes,
                         "bytes_per_node_sample": bpns, "peak_source": peak_src,
                         "traffic_source": traffic_src, "sweep_share_of_step": sw / ms,
                         "timing": ("external events around the sweep node inside the replayed step graph, "
                                    "L2 flushed before each step" if floor_ms is not None else
                                    "events around the sweep launch in eager visits, L2 flushed"),
                         "event_floor_ms": floor_ms,
                         "frac_above_event_floor": (algo_bytes / ((sw - floor_ms) * 1e-3) / 1e9 / peak
                                                    if floor_ms is not None and sw > floor_ms else None),
                         "limiter": ("instruction issue (ALU pipe: Philox, alias draws, tally), not HBM: "
                                     "see DESIGN.md 6" if eng.joint else
                                     "instruction issue (Philox + table draws), not HBM: see DESIGN.md 6")},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(host_obs.numel()),
                    "host_format": (f"{graphs.obs_bits}-bit .sgb block" if graphs is not None and graphs.nibbles
                                    else "int8 block"),
                    "d2h_bytes_per_step": eng.pack.cells * 8, "ms_per_step": e2e_ms,
                    "mode": ("the C2 minibatch (moving sum, lanes resident) re-uploaded from pinned memory and "
                             "range-checked every step, CPTs read back every step; `--workload c2s` streams "
                             "different minibatches that each step samples"),
                    "launch": (f"{per_call} visits per graph replay, uploads on a copy stream"
                               if e2e_graphs is not None else "eager visits"),
                    # the step's upload against the link: the e2e step is PCIe-bound when this nears the best rate
                    "h2d_gbs": host_obs.numel() * host_obs.element_size() / (e2e_ms * 1e-3) / 1e9,
                    "host_enqueue_us_per_step": host_enqueue_us, "h2d_warmup": h2d_warm},
            "gpu_launches": launches,
            "launch_mode": "cuda-graph replay per step" if graphs is not None else "eager",
            "kernel_path": ("packed-lane sg_joint_sweep + merged step tail (sg_step_tail_joint)" if eng.joint else
                            "packed-lane sg_small_sweep + sg_step_finish" if eng.use_small else
                            "device site keys + sg_np_uniforms + generic sg_sweep (injected) + sg_step_finish"
                            if eng.rng_mode == _lib.SG_RNG_NUMPY else "generic sg_sweep + sg_step_finish"),
            "clocks": clk.summary(),
        }
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(wl, n_vars)
        print(json.dumps(out))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def stream_arm(args, wl: Workload) -> None:
    """C5: a pass over an on-disk 4-bit .sgb file of ``--c5-cases`` cases per GPU
    (default 10^7), streamed through BinaryFileSource: disk -> pinned buffer ->
    device on a copy stream one minibatch ahead, decoded on the device.  The
    timed region is the whole pass (every minibatch of the file, after a
    separate warm-up pass over the first ``--warmup`` blocks); a step is one
    minibatch visit."""
    import tempfile

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1511_06416_b200 as sg
    from paper_1511_06416_b200 import _lib, io
    from paper_1511_06416_b200.engine import Engine

    B, M = wl.cases, wl.m
    cases = int(args.c5_cases)
    net, truth = wl.network()
    n_vars = net.num_vars
    base = rank * cases  # this rank's shard of the global data set
    tmpdir = tempfile.mkdtemp(prefix="sg_c5_", dir=os.environ.get("SG_C5_DIR") or None)
    path = os.path.join(tmpdir, f"c5_rank{rank}.sgb")
    latent_cells = [0, 0]

    def block(lo, hi):
        obs = sg.forward_sample_device(net, truth, hi - lo, seed=105, hide_fraction=0.3, mask_seed=205,
                                       case_base=base + lo)[:, :hi - lo]
        latent_cells[0] += int((obs < 0).sum())
        latent_cells[1] += obs.numel()
        return obs

    t_w = time.perf_counter()
    io.write_binary_blocks(path, n_vars, cases, B, block, "nibble")
    write_s = time.perf_counter() - t_w
    latent = latent_cells[0] / max(1, latent_cells[1])
    src = io.BinaryFileSource(path)
    nblocks = (cases + B - 1) // B
    if args.rng == "auto":
        args.rng = "fast"  # DAG-1000: no packed lane word
    cfg = sg.SamplerConfig(same_m=M, minibatch_size=B, num_passes=1, seed=300, rng=args.rng,
                           accumulator_mode="exponential", exp_decay=0.9)
    comm = (lambda c: dist.all_reduce(c)) if world > 1 else None
    eng = Engine(net, cfg, case_base=base, comm=comm)
    for k, mb in enumerate(src):  # warm-up: the first blocks of the file
        if k >= args.warmup:
            break
        eng.visit(mb, 0, M)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(nblocks + 1)]
    launches0 = _lib.launch_count
    h0 = time.perf_counter()
    with ClockSampler(local) as clk:
        marks[0].record()
        for k, mb in enumerate(src):  # the whole file: every step's block is read, uploaded and decoded
            eng.visit(mb, 1, M)
            marks[k + 1].record()
        torch.cuda.synchronize()
    wall = time.perf_counter() - h0
    launches = _lib.launch_count - launches0
    if eng.err.read():
        raise RuntimeError("device error word set")
    ms = marks[0].elapsed_time(marks[nblocks]) / nblocks  # reads + copies + visits, back to back
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
    node_samples = n_vars * cases * M / nblocks  # per GPU per step (mean over the pass)
    value = world * node_samples / (ms * 1e-3)
    h2d = n_vars * src.header["pitch"] // 2  # 4-bit block bytes per step
    if rank == 0:
        try:
            peak = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
        except Exception:  # noqa: BLE001
            peak = 6650.0
        bpns = 1.0 + latent
        hbm_gbs = bpns * node_samples / (ms * 1e-3) / 1e9
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": nblocks,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int8 states, u32 draws, f64 CPTs", "data": "synthetic",
            "config": dict(wl.config(world, args.rng, n_vars), latent_fraction=round(latent, 4),
                           cases_per_gpu=cases, file=f"4-bit .sgb, {os.path.getsize(path) / 1e9:.2f} GB per GPU",
                           l2="inputs stream from disk / host memory every step"),
            "roofline": {"bound": "hbm", "achieved": hbm_gbs, "peak": peak, "unit": "GB/s", "frac": hbm_gbs / peak,
                         "traffic": None, "note": "whole step (sweep + tally + tail + decode), algorithmic bytes "
                                                   "n x B x m x (1 + f) per step"},
            "pcie": {"h2d_gbs": h2d / (ms * 1e-3) / 1e9, "h2d_bytes_per_step": h2d,
                     "frac_of_50gbs": h2d / (ms * 1e-3) / 50e9},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 0,
                    "note": "value is already end to end: every step's minibatch is read from the .sgb file, "
                            "copied from pinned host memory and decoded on the device"},
            "gpu_launches": launches, "launch_mode": "eager, copy stream one minibatch ahead",
            "kernel_path": "BinaryFileSource + sg_unpack_nibbles + generic big-tile sweep + chunked tally + step tail",
            "file_write_s": round(write_s, 1), "pass_wall_s": round(wall, 2), "clocks": clk.summary(),
        }
        print(json.dumps(out))
    try:
        os.remove(path)
        os.rmdir(tmpdir)
    except OSError:
        pass
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def stream_small_arm(args, wl: Workload) -> None:
    """C2 streamed (``--workload c2s``): the Koller workload of C2 (m = 10, 1M-case
    minibatches, 50 % hidden, joint stream) over ``--c2s-cases`` cases per GPU
    (default 10^8) held as 2-bit .sgb blocks in pinned host memory, driven
    through the public API: ``run(net, HostSource(...), cfg)`` with the
    exponential accumulator, i.e. every step copies its minibatch host ->
    device, decodes it and replays a stream graph (prepare + sweep + tail)
    that samples it.  Two passes; the second (pure steady state: graph
    capture and the first eager visit are in pass 1) is reported, timed by
    run()'s own per-pass CUDA events."""
    import torch

    import paper_1511_06416_b200 as sg
    from paper_1511_06416_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:  # independent replicas: every rank streams its own shard, no collective in this line
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    B, M = 1_000_000, 10
    cases = int(args.c2s_cases)
    net, truth = WORKLOADS["c2"].network()
    base = rank * cases
    t0 = time.perf_counter()
    src = sg.HostSource.from_device_blocks(
        lambda lo, hi: sg.forward_sample_device(net, truth, hi - lo, seed=100, hide_fraction=0.5, mask_seed=200,
                                                case_base=base + lo)[:, :hi - lo], net.num_vars, cases, B, bits=2)
    build_s = time.perf_counter() - t0
    cfg = sg.SamplerConfig(same_m=M, minibatch_size=B, num_passes=2, seed=300, rng="joint",
                           accumulator_mode="exponential", exp_decay=0.9)
    launches0 = _lib.launch_count
    with ClockSampler(local) as clk:
        _, trace = sg.run(net, src, cfg, engine_hook=lambda e: setattr(e, "case_base", base))
    launches = _lib.launch_count - launches0
    rec = trace.records[1]
    secs = rec.seconds - trace.records[0].seconds
    steps = (cases + B - 1) // B
    value = world * rec.vars_sampled / secs
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([secs], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        value = world * rec.vars_sampled / float(t[0])
        dist.destroy_process_group()
    if rank == 0:
        h2d = net.num_vars * max(64, (B + 63) // 64 * 64) // 4
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps, "warmup": steps,
            "ms_per_step": secs / steps * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "int8 states, u32 draws, f64 CPTs", "data": "synthetic",
            "config": {"workload": f"C2 streamed: koller-student, {cases} cases per GPU as 2-bit .sgb blocks in pinned "
                                   "host memory, minibatch 1M, SAME m=10, 50% hidden, exponential accumulator "
                                   "(decay 0.9), rng=joint, pass 2 of 2 reported",
                       "network": "koller-student", "cases_per_gpu": cases, "m": M, "rng": "joint",
                       "api": "run(net, HostSource.from_device_blocks(..., bits=2), cfg)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 0,
                    "note": "already end to end: every step's minibatch is copied from pinned host memory, decoded "
                            "and sampled; CPTs stay on the device until the end of the run"},
            "pcie": {"h2d_gbs": h2d / (secs / steps) / 1e9},
            "gpu_launches": launches, "launch_mode": "stream graphs (one replay per minibatch)",
            "host_blocks_build_s": round(build_s, 1), "clocks": clk.summary(),
        }
        print(json.dumps(out))


def main() -> None:
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS) + ["c2s"], default="c2")
    ap.add_argument("--rng", choices=["auto", "joint", "fast", "numpy"], default="auto",
                    help="auto: joint (one draw per lane per sweep) when the network's lane word fits, else fast")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--eager", action="store_true", help="launch each visit eagerly instead of graph replay")
    ap.add_argument("--c5-cases", type=int, default=10_000_000, help="C5: cases per GPU in the streamed .sgb file")
    ap.add_argument("--c2s-cases", type=int, default=100_000_000, help="c2s: cases per GPU streamed from host memory")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        # communicator set-up lines (rank / nranks, NVLS, rings) on stderr, so a
        # multi-GPU line can be checked against the ranks NCCL actually formed
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    if args.workload == "c2s":
        if args.impl == "reference":
            args.workload = "c2"  # the reference arm of the same C2 workload
        else:
            stream_small_arm(args, None)
            return
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        reference_arm(args, wl)
    elif wl.key == "c5":
        stream_arm(args, wl)
    else:
        our_arm(args, wl)


if __name__ == "__main__":
    main()

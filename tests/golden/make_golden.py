"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (the reference is importable there, read-only):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports samegibbs from /root/reference/pkg/src, runs the reference's own
functions on small seeded inputs and stores inputs and outputs as .npz files
next to this script.  The fixtures travel with the repo; the reference does
not (nothing at test time reads /root/reference).

Fixtures:
  sweep_*.npz    one reference sweep: CPTs, lane values before/after, latent
                 lane lists, lane weights, per-variable uniforms it consumed
                 (recorded through a substream shim), count tables
  init_*.npz     reference init_latent on a replicated batch
  run_*.npz      reference run(): final CPTs and per-pass kl_avg (MAP mode is
                 a deterministic function of the uniforms, so it is bit-exact)
  data_koller.npz  reference forward_sample + mask (dense)
  rng.npz        blake2b site keys and numpy Philox draws
  mean_cpts.npz  reference mean_cpts on count tables with card 2..12
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.dont_write_bytecode = True
sys.path.insert(0, str(REF))
sys.path.insert(0, str(REF.parent / "tests"))

import samegibbs  # noqa: E402
from samegibbs import (DirichletPrior, SamplerConfig, build_network, color_graph, forward_sample,  # noqa: E402
                       init_cpts, mask, moralize, run)
from samegibbs import sampler as ref_sampler  # noqa: E402
from samegibbs.io import bundled_network_path, load_network_file  # noqa: E402
from samegibbs.model import mean_cpts, tally_counts  # noqa: E402
from samegibbs.rng import derive_seed, stream_key, substream  # noqa: E402
from samegibbs.sampler import init_latent, pad_block, replicate_minibatch, sweep  # noqa: E402


def tables_to(prefix, tables, d):
    for i, t in enumerate(tables):
        d[f"{prefix}_{i}"] = np.asarray(t)


def net_to(net, d):
    d["cards"] = np.asarray(net.cardinalities, dtype=np.int64)
    d["edges"] = np.asarray([(p, c) for c in range(net.num_vars) for p in net.parents[c]],
                            dtype=np.int64).reshape(-1, 2)


class Recorder:
    """substream shim: records every .random(k) draw of the "var" sites."""

    def __init__(self):
        self.log = {}

    def __call__(self, seed, label, *idx):
        gen = substream(seed, label, *idx)
        if label != "var":
            return gen
        rec = self

        class Proxy:
            def random(self, k):
                u = gen.random(k)
                rec.log[idx[0]] = u.copy()
                return u

        return Proxy()


def sweep_fixture(name, net, cpts, dense, m, init_seed, sweep_seed, real=None):
    real = dense.shape[1] if real is None else real
    mb = pad_block(0, dense[:, :real].astype(np.int32), dense.shape[1])
    batch = replicate_minibatch(mb, m)
    init_latent(net, batch, init_seed, 0, 0)
    before = batch.values.copy()
    coloring = color_graph(moralize(net))
    rec = Recorder()
    orig = ref_sampler.substream
    ref_sampler.substream = rec
    try:
        counts = sweep(net, coloring, cpts, batch, sweep_seed)
    finally:
        ref_sampler.substream = orig
    d = {"m": np.int64(m), "base_size": np.int64(dense.shape[1]), "num_real": np.int64(real),
         "sweep_seed": np.uint64(sweep_seed), "before": before, "after": batch.values.copy(),
         "weights": batch.lane_weights.copy()}
    net_to(net, d)
    tables_to("cpt", cpts.tables, d)
    tables_to("counts", counts.tables, d)
    for v in range(net.num_vars):
        d[f"missing_{v}"] = batch.missing_lanes[v]
        d[f"u_{v}"] = rec.log.get(v, np.zeros(0))
    d["groups"] = np.asarray([g for grp in coloring.groups for g in grp] , dtype=np.int64)
    d["group_sizes"] = np.asarray([len(g) for g in coloring.groups], dtype=np.int64)
    np.savez_compressed(OUT / f"sweep_{name}.npz", **d)


def main():
    os.chdir(OUT)
    koller, truth = load_network_file(bundled_network_path("koller"))

    # --- sweeps on the Koller network
    data = mask(forward_sample(koller, truth, 500, seed=1), 0.5, seed=2)
    dense = data.to_dense()
    sweep_fixture("koller_m3", koller, truth, dense, 3, 7, derive_seed(11, "sweep", 0, 0, 0))
    sweep_fixture("koller_pad", koller, init_cpts(koller, 5), dense[:, :96], 2, 8, 12345, real=70)

    # --- random networks (helpers.random_network, cards up to 4; one with large cards)
    from helpers import random_cpts, random_network

    rng = np.random.default_rng(2024)
    for k in range(4):
        net = random_network(rng, int(rng.integers(4, 9)), 0.4, max_card=4)
        cp = random_cpts(net, rng, concentration=1.5)
        d = forward_sample(net, cp, 200, seed=30 + k)
        dd = mask(d, 0.45, seed=40 + k).to_dense()
        sweep_fixture(f"rand{k}", net, cp, dd, 1 + k, 50 + k, 60 + k)
    big = build_network([9, 12, 3, 8, 2], [(0, 1), (0, 2), (1, 2), (2, 3), (1, 4), (3, 4)])
    cp = random_cpts(big, rng, concentration=0.7)
    dd = mask(forward_sample(big, cp, 150, seed=71), 0.6, seed=72).to_dense()
    sweep_fixture("bigcard", big, cp, dd, 2, 73, 74)

    # --- larger shapes of BASELINE configs C3/C4 (generators: paper_1511_06416_b200/netgen.py)
    sys.path.insert(0, str(OUT.parents[1]))
    from paper_1511_06416_b200 import netgen

    def ref_net(n):
        return build_network(list(n.cardinalities), [(p, c) for c in range(n.num_vars) for p in n.parents[c]])

    dag = ref_net(netgen.random_dag_network(120, max_parents=4, min_card=2, max_card=4, seed=11))
    cp = random_cpts(dag, np.random.default_rng(12), concentration=0.8)
    dd = mask(forward_sample(dag, cp, 160, seed=13), 0.3, seed=14).to_dense()
    sweep_fixture("dag120", dag, cp, dd, 2, 15, 16)
    mooc = ref_net(netgen.mooc_network(10, 60, seed=3))
    cp = random_cpts(mooc, np.random.default_rng(4), concentration=1.0)
    dd = mask(forward_sample(mooc, cp, 150, seed=5), 0.7, seed=6).to_dense()
    dd[:10] = -1  # concepts are never observed
    sweep_fixture("mooc", mooc, cp, dd, 5, 7, 8)

    # --- init_latent
    mb = pad_block(0, dense[:, :64].astype(np.int32), 64)
    batch = replicate_minibatch(mb, 4)
    init_latent(koller, batch, 99, 3, 1)
    d = {"values": batch.values, "seed": np.int64(99), "context": np.asarray([3, 1]), "m": np.int64(4),
         "dense": dense[:, :64]}
    np.savez_compressed(OUT / "init_koller.npz", **d)

    # --- run(): MAP (bit-exact) and sampled (statistical)
    data600 = mask(forward_sample(koller, truth, 600, seed=21), 0.5, seed=22)
    dense600 = data600.to_dense()
    runs = {
        "map_moving": SamplerConfig(same_m=2, minibatch_size=100, num_passes=3, map_estimate=True, seed=4),
        "map_exp": SamplerConfig(same_m=3, minibatch_size=128, num_passes=2, map_estimate=True, seed=5,
                                 accumulator_mode="exponential", exp_decay=0.7),
        "map_sweeps2": SamplerConfig(same_m=[(1, 1), (2, 2)], minibatch_size=150, num_passes=3,
                                     map_estimate=True, seed=6, sweeps_per_minibatch=2),
        "sampled": SamplerConfig(same_m=5, minibatch_size=200, num_passes=20, seed=7),
    }
    for name, cfg in runs.items():
        cpts, trace = run(koller, data600, cfg, truth=truth)
        d = {"dense": dense600, "kl": np.asarray([r.kl_avg for r in trace.records]),
             "vars_sampled": np.asarray([r.vars_sampled for r in trace.records])}
        tables_to("cpt", cpts.tables, d)
        tables_to("truth", truth.tables, d)
        np.savez_compressed(OUT / f"run_{name}.npz", **d)

    # --- data generation
    full = forward_sample(koller, truth, 300, seed=100).to_dense()
    masked = mask(forward_sample(koller, truth, 300, seed=100), 0.5, seed=200).to_dense()
    np.savez_compressed(OUT / "data_koller.npz", full=full, masked=masked)

    # --- RNG sites and streams
    labels = [(0, "sweep", (0, 0, 0)), (300, "var", (4,)), (123456789, "latent_init", (2, 7, 1)),
              (2**63 + 5, "cpt_update", (1, 2))]
    keys = np.asarray([stream_key(s, l, *i) for s, l, i in labels], dtype=np.uint64)
    draws = np.stack([substream(s, l, *i).random(17) for s, l, i in labels])
    ints = np.stack([substream(s, l, *i).integers(0, 3, size=40, dtype=np.int32) for s, l, i in labels])
    big_ints = np.stack([substream(s, l, *i).integers(0, 2**30 + 1, size=40, dtype=np.int32) for s, l, i in labels])
    np.savez_compressed(OUT / "rng.npz", keys=keys, draws=draws, ints=ints, big_ints=big_ints,
                        seeds=np.asarray([s for s, _, _ in labels], dtype=np.uint64),
                        labels=np.asarray([l for _, l, _ in labels]),
                        idx=np.asarray([",".join(map(str, i)) for _, _, i in labels]))

    # --- mean_cpts with cards 2..12 (pairwise row sums for card >= 8)
    mnet = build_network([2, 12, 9, 8, 3], [(0, 1), (1, 2), (0, 3), (3, 4)])
    crng = np.random.default_rng(5)
    counts = samegibbs.CountSet([crng.integers(0, 50, size=mnet.table_shape(i)).astype(np.float64)
                                 for i in range(mnet.num_vars)])
    prior = DirichletPrior(0.3, per_variable=(0.3, 1.0, 0.01, 2.5, 1e-6))
    out = mean_cpts(counts, prior)
    d = {"alphas": np.asarray(prior.per_variable)}
    net_to(mnet, d)
    tables_to("counts", counts.tables, d)
    tables_to("mean", out.tables, d)
    # tally of random complete assignments with 0/1 weights
    vals = np.stack([crng.integers(0, c, size=300) for c in mnet.cardinalities]).astype(np.int32)
    w = (crng.random(300) < 0.8).astype(np.float64)
    tab = tally_counts(mnet, vals, w)
    d["tally_values"] = vals
    d["tally_weights"] = w
    tables_to("tally", tab.tables, d)
    np.savez_compressed(OUT / "model.npz", **d)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()

"""Acceptance-protocol fixtures made by running the REFERENCE (statistical parity anchors).

Run in the build container (the reference is importable there, read-only):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_acceptance.py [--skip-c2]
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_acceptance.py --spread

Fixtures written next to this script:

  accept_koller.npz   the reference's Koller protocol (test_acceptance.py:46-97):
                      50k cases (forward_sample seed 100+s, mask 0.5 seed 200+s),
                      minibatch 12,500, 200 passes, sampler seed 300+s, for
                      m in (1, 5, 10) x s in 0..4.  Stores the final kl_avg,
                      avg_abs_error, the per-pass kl trace and the final CPTs
                      of each of the 15 runs.
  accept_c2.npz       the reference at the bench configuration C2 (BASELINE
                      configs[1]): Koller, 1,000,000 cases (forward_sample
                      seed 100, mask 0.5 seed 200), SAME m = 10, one minibatch
                      of 1M, moving sum, sampled Dirichlet, 12 passes, sampler
                      seeds 300, 301, 302 (the reference's own run-to-run
                      spread).  Per-pass kl trace and final CPTs per seed.
  accept_seeds.npz    the sampler's own spread: the protocol's data of seed 0,
                      m in (1, 10), sampler seeds 300..323 (24 reference runs
                      per m): final kl_avg and avg_abs_error of each run.
  predict_c10.npz     reference predict_missing (metrics.py:89-139) on the c10
                      network (test_acceptance.py:287-306) with the generating
                      CPTs frozen: context, targets, 40 kept sweeps after 5
                      burn-in, frequencies (numpy RNG: bit-exact target), plus
                      the reference's c10 AUCs after 10 and 100 passes.

Runs in parallel processes (one reference run per process).
"""

from __future__ import annotations

import os
import sys
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.dont_write_bytecode = True
sys.path.insert(0, str(REF))
sys.path.insert(0, str(REF.parent / "tests"))

PROTOCOL = dict(minibatch_size=12_500, num_passes=200)
C2_CASES, C2_M, C2_PASSES, C2_SEEDS = 1_000_000, 10, 12, (300, 301, 302)


def _koller():
    from samegibbs.io import bundled_network_path, load_network_file

    return load_network_file(bundled_network_path("koller"))


def koller_protocol(args):
    m, seed = args
    from samegibbs import SamplerConfig, avg_abs_error, forward_sample, kl_avg, mask, run

    net, truth = _koller()
    data = mask(forward_sample(net, truth, 50_000, seed=100 + seed), 0.5, seed=200 + seed)
    cfg = SamplerConfig(same_m=m, seed=300 + seed, **PROTOCOL)
    cpts, trace = run(net, data, cfg, truth=truth)
    return (m, seed, [r.kl_avg for r in trace.records], avg_abs_error(truth, cpts), kl_avg(truth, cpts),
            [np.asarray(t) for t in cpts.tables])


SPREAD_SEEDS = tuple(range(300, 324))


def koller_spread(args):
    m, sampler_seed = args
    from samegibbs import SamplerConfig, avg_abs_error, forward_sample, kl_avg, mask, run

    net, truth = _koller()
    data = mask(forward_sample(net, truth, 50_000, seed=100), 0.5, seed=200)
    cfg = SamplerConfig(same_m=m, seed=sampler_seed, **PROTOCOL)
    cpts, _ = run(net, data, cfg, truth=truth)
    return m, sampler_seed, kl_avg(truth, cpts), avg_abs_error(truth, cpts)


def c2_run(seed):
    from samegibbs import SamplerConfig, avg_abs_error, forward_sample, mask, run

    net, truth = _koller()
    data = mask(forward_sample(net, truth, C2_CASES, seed=100), 0.5, seed=200)
    cfg = SamplerConfig(same_m=C2_M, minibatch_size=C2_CASES, num_passes=C2_PASSES, seed=seed)
    cpts, trace = run(net, data, cfg, truth=truth)
    return seed, [r.kl_avg for r in trace.records], avg_abs_error(truth, cpts), [np.asarray(t) for t in cpts.tables]


def c10_predict(_=None):
    from helpers import random_cpts, random_network
    from samegibbs import SamplerConfig, forward_sample, mask, predict_missing, roc_auc, run, train_test_split

    rng = np.random.default_rng(4242)
    net = random_network(rng, 20, 0.12, max_card=2)
    truth = random_cpts(net, rng)
    full = forward_sample(net, truth, 4000, seed=11)
    sparse = mask(full, 0.9, seed=12)
    train_set, test_set = train_test_split(sparse, 0.8, seed=13)
    targets = np.asarray(list(zip(test_set.var_idx.tolist(), test_set.case_idx.tolist())), dtype=np.int64)
    labels = test_set.values.astype(np.int64)
    freq = predict_missing(net, truth, train_set, [tuple(t) for t in targets], num_samples=40, seed=15, burn_in=5)
    aucs = []
    for passes in (10, 100):
        cfg = SamplerConfig(minibatch_size=2000, num_passes=passes, seed=14)
        cpts, _ = run(net, train_set, cfg)
        probs = predict_missing(net, cpts, train_set, [tuple(t) for t in targets], num_samples=300, seed=15,
                                burn_in=30)
        aucs.append(roc_auc(probs[:, 1], labels).auc)
    d = {"cards": np.asarray(net.cardinalities, dtype=np.int64),
         "edges": np.asarray([(p, c) for c in range(net.num_vars) for p in net.parents[c]],
                             dtype=np.int64).reshape(-1, 2),
         "context": train_set.to_dense(), "targets": targets, "labels": labels, "freq": freq,
         "num_samples": np.int64(40), "burn_in": np.int64(5), "seed": np.int64(15),
         "auc_10": np.float64(aucs[0]), "auc_100": np.float64(aucs[1])}
    for i, t in enumerate(truth.tables):
        d[f"cpt_{i}"] = np.asarray(t)
    return d


def spread_main():
    jobs = [(m, s) for m in (1, 10) for s in SPREAD_SEEDS]
    with ProcessPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        res = list(ex.map(koller_spread, jobs))
    d = {"ms": np.asarray([r[0] for r in res]), "seeds": np.asarray([r[1] for r in res]),
         "kl": np.asarray([r[2] for r in res]), "abs_err": np.asarray([r[3] for r in res])}
    np.savez_compressed(OUT / "accept_seeds.npz", **d)
    print("accept_seeds.npz: mean kl by m", {m: float(d["kl"][d["ms"] == m].mean()) for m in (1, 10)}, flush=True)


def main():
    if "--spread" in sys.argv:
        spread_main()
        return
    skip_c2 = "--skip-c2" in sys.argv
    jobs = [(m, s) for m in (1, 5, 10) for s in range(5)]
    with ProcessPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        c2f = [] if skip_c2 else [ex.submit(c2_run, s) for s in C2_SEEDS]
        pf = ex.submit(c10_predict)
        res = list(ex.map(koller_protocol, jobs))
        d = {"ms": np.asarray([r[0] for r in res]), "seeds": np.asarray([r[1] for r in res]),
             "kl_trace": np.asarray([r[2] for r in res]), "abs_err": np.asarray([r[3] for r in res]),
             "kl": np.asarray([r[4] for r in res])}
        for i, r in enumerate(res):
            for v, t in enumerate(r[5]):
                d[f"cpt_{i}_{v}"] = t
        np.savez_compressed(OUT / "accept_koller.npz", **d)
        print("accept_koller.npz: median kl by m",
              {m: float(np.median(d["kl"][d["ms"] == m])) for m in (1, 5, 10)}, flush=True)
        np.savez_compressed(OUT / "predict_c10.npz", **pf.result())
        print("predict_c10.npz written", flush=True)
        if c2f:
            c2 = [f.result() for f in c2f]
            d = {"seeds": np.asarray([r[0] for r in c2]), "kl_trace": np.asarray([r[1] for r in c2]),
                 "abs_err": np.asarray([r[2] for r in c2]), "cases": np.int64(C2_CASES), "m": np.int64(C2_M),
                 "passes": np.int64(C2_PASSES)}
            for i, r in enumerate(c2):
                for v, t in enumerate(r[3]):
                    d[f"cpt_{i}_{v}"] = t
            np.savez_compressed(OUT / "accept_c2.npz", **d)
            print("accept_c2.npz: final kl", d["kl_trace"][:, -1], flush=True)


if __name__ == "__main__":
    main()

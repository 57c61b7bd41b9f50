"""Synthetic network shapes of the BASELINE.json workloads C3-C5.

The reference ships one network (Koller's student network, data/koller.json)
and, in its test helpers, a random-DAG generator (tests/helpers.py:19-35,
edge probability per ordered pair).  BASELINE.json names two more shapes,
built here deterministically from a seed:

* :func:`random_dag_network` -- C4/C5: ``n`` nodes in a random topological
  order, node ``i`` of the order draws its in-degree uniformly from
  ``0..min(max_parents, i)`` and its parents uniformly among earlier nodes;
  cardinalities uniform in ``[min_card, max_card]``.
* :func:`mooc_network` -- C3: binary latent concepts (each with up to three
  concept parents) and binary/ternary questions hanging off one to three
  concepts (mostly one, so the CPT has a few hundred rows per hundred
  questions).  :func:`mooc_observations` hides every concept and keeps a
  sparse fraction of the question responses.
* :func:`dirichlet_cpts` -- generating CPTs with Dirichlet rows
  (tests/helpers.py:38-43).

These are workload generators (host, once per run); the sweep never calls
them.
"""

from __future__ import annotations

import numpy as np
import torch

from .model import CptSet
from .network import Network, build_network


def random_dag_network(num_vars: int, max_parents: int = 4, min_card: int = 2, max_card: int = 4,
                       seed: int = 0) -> Network:
    """Random DAG with in-degree <= max_parents (C4: 1000 nodes, in-degree <= 4, cards 2-4)."""
    rng = np.random.default_rng(seed)
    cards = [int(c) for c in rng.integers(min_card, max_card + 1, size=num_vars)]
    order = rng.permutation(num_vars)
    edges = []
    for i in range(1, num_vars):
        k = int(rng.integers(0, min(max_parents, i) + 1))
        if k:
            for j in rng.choice(i, size=k, replace=False):
                edges.append((int(order[j]), int(order[i])))
    return build_network(cards, edges)


def mooc_network(num_concepts: int = 15, num_questions: int = 319, ternary_fraction: float = 0.2,
                 seed: int = 0) -> Network:
    """Student/concept/question network (C3).  Variables 0..num_concepts-1 are
    the binary concepts (concept i takes 0..min(3, i) earlier concepts as
    parents); the rest are questions with 1, 2 or 3 concept parents
    (probabilities 0.9 / 0.08 / 0.02) and 2 or 3 states."""
    rng = np.random.default_rng(seed)
    cards = [2] * num_concepts
    edges = []
    for i in range(1, num_concepts):
        k = int(rng.integers(0, min(3, i) + 1))
        for j in rng.choice(i, size=k, replace=False):
            edges.append((int(j), i))
    for q in range(num_questions):
        v = num_concepts + q
        cards.append(3 if rng.random() < ternary_fraction else 2)
        k = int(rng.choice([1, 2, 3], p=[0.9, 0.08, 0.02]))
        for j in rng.choice(num_concepts, size=min(k, num_concepts), replace=False):
            edges.append((int(j), v))
    return build_network(cards, edges)


def dirichlet_cpts(net: Network, concentration: float = 1.0, seed: int = 0) -> CptSet:
    """Generating CPTs: every row ~ Dirichlet(concentration) (tests/helpers.py:38-43)."""
    rng = np.random.default_rng(seed)
    tables = []
    for v in range(net.num_vars):
        rows, card = net.table_shape(v)
        tables.append(rng.dirichlet(np.full(card, concentration), size=rows))
    return CptSet(tables)


def mooc_observations(net: Network, cpts: CptSet, num_cases: int, num_concepts: int, density: float,
                      seed: int, case_base: int = 0) -> torch.Tensor:
    """Device int8 (n, ld) matrix of C3: complete cases forward-sampled with the
    reference's streams, every concept hidden, each question response kept with
    probability ``density`` (mask stream of ``seed + 1``)."""
    from .datagen import forward_sample_device

    full = forward_sample_device(net, cpts, num_cases, seed=seed, case_base=case_base)
    gen = torch.Generator(device=full.device)
    gen.manual_seed(seed + 1 + case_base)
    keep = torch.rand(full.shape, generator=gen, device=full.device) < density
    out = torch.where(keep, full, torch.full_like(full, -1))
    out[:num_concepts] = -1
    out[:, num_cases:] = -1
    return out

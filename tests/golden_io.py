"""Loading helpers for the reference-generated fixtures in tests/golden/."""

from __future__ import annotations

from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def load(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz", allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def tables(d: dict, prefix: str) -> list:
    out, i = [], 0
    while f"{prefix}_{i}" in d:
        out.append(d[f"{prefix}_{i}"])
        i += 1
    return out


def per_var(d: dict, prefix: str, n: int) -> list:
    return [d[f"{prefix}_{v}"] for v in range(n)]


def edges(d: dict) -> list:
    return [tuple(int(x) for x in e) for e in d["edges"]]


SWEEPS = ["koller_m3", "koller_pad", "rand0", "rand1", "rand2", "rand3", "bigcard", "dag120", "mooc"]
RUNS_MAP = ["map_moving", "map_exp", "map_sweeps2"]

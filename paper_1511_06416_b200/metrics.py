"""Evaluation helpers of the reference API (``samegibbs/metrics.py``).

``kl_avg`` / ``avg_abs_error`` / ``roc_auc`` / ``throughput`` are host-side
reductions over model-sized tables or score lists (evaluation, not the sweep).
``predict_missing`` reuses the device sweep with frozen CPTs.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np

from .errors import DegenerateLabels, DimensionMismatch, EmptyTrace
from .model import CptSet, check_congruent


def kl_avg(truth: CptSet, estimate: CptSet) -> float:
    """Mean over CPT rows of sum_x p ln(p/q), skipping q = 0 terms (metrics.py:19-37)."""
    check_congruent(truth, estimate)
    total, rows = 0.0, 0
    for p, q in zip(truth.tables, estimate.tables):
        keep = (p > 0) & (q > 0)
        with np.errstate(divide="ignore", invalid="ignore"):
            total += float(np.where(keep, p * np.log(p / q), 0.0).sum())
        rows += p.shape[0]
    return total / rows


def avg_abs_error(truth: CptSet, estimate: CptSet) -> float:
    """Mean |p - q| over all CPT cells (metrics.py:40-45)."""
    check_congruent(truth, estimate)
    cells = sum(p.size for p in truth.tables)
    return sum(float(np.abs(p - q).sum()) for p, q in zip(truth.tables, estimate.tables)) / cells


@dataclass
class RocCurve:
    points: np.ndarray
    auc: float


def roc_auc(scores: Sequence[float], labels: Sequence[int]) -> RocCurve:
    """ROC with tied scores as one step; trapezoid AUC = Mann-Whitney (metrics.py:56-86)."""
    s = np.asarray(scores, dtype=np.float64)
    y = np.asarray(labels, dtype=np.int64)
    if s.shape != y.shape:
        raise DimensionMismatch("scores and labels differ in length")
    pos = int((y == 1).sum())
    neg = int((y == 0).sum())
    if pos == 0 or neg == 0:
        raise DegenerateLabels("need both positive and negative labels")
    order = np.argsort(-s, kind="mergesort")
    s, y = s[order], y[order]
    last = np.r_[np.flatnonzero(np.diff(s) != 0), len(s) - 1]
    tp = np.r_[0, np.cumsum(y == 1)[last]].astype(np.float64)
    fp = np.r_[0, np.cumsum(y == 0)[last]].astype(np.float64)
    area2 = float(np.sum((fp[1:] - fp[:-1]) * (tp[1:] + tp[:-1])))
    return RocCurve(points=np.column_stack([fp / neg, tp / pos]), auc=area2 / (2.0 * pos * neg))


@dataclass
class ThroughputSummary:
    per_pass: list
    overall: float | None


def throughput(trace) -> ThroughputSummary:
    """Node-samples per second per pass and overall (metrics.py:150-163)."""
    if not trace.records:
        raise EmptyTrace("trace has no records")
    per, prev = [], 0.0
    for r in trace.records:
        dt = r.seconds - prev
        per.append(r.vars_sampled / dt if dt > 0 else None)
        prev = r.seconds
    tot = trace.records[-1].seconds
    return ThroughputSummary(per_pass=per,
                             overall=sum(r.vars_sampled for r in trace.records) / tot if tot > 0 else None)


def predict_missing(net, cpts: CptSet, context, targets, num_samples: int, seed: int,
                    burn_in: int = 0) -> np.ndarray:
    """Per-target state frequencies under frozen CPTs (metrics.py:89-139), device sweeps."""
    from .predict import predict_missing as _pm

    return _pm(net, cpts, context, targets, num_samples, seed, burn_in)

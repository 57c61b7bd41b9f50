"""Held-out prediction with frozen CPTs (reference ``metrics.predict_missing``,
metrics.py:89-139), on the device.

The context's present entries stay clamped; every other cell is latent and is
resampled by ``burn_in + num_samples`` sweeps keyed ``derive_seed(seed,
"predict", it)`` (numpy RNG mode, so the result is bit-identical to the
reference).  The latent init is ``(seed, "latent_init", 0)`` as in the
reference.  Site keys are hashed on the device (``sg_site_keys``) and the
target frequencies are tallied by ``sg_predict_tally`` after each kept sweep
(the reference's ``np.add.at``, metrics.py:136-137); one host sync at the end.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .device import ErrorWord, device, netpack, stream_handle, var_keys
from .errors import DimensionMismatch, ValidationError
from .network import color_graph, moralize
from .rng import derive_seed
from .sampler import DeviceBatch, _raise_errors


def predict_missing(net, cpts, context, targets, num_samples: int, seed: int, burn_in: int = 0) -> np.ndarray:
    if context.num_vars != net.num_vars:
        raise DimensionMismatch(f"context has {context.num_vars} variables, network has {net.num_vars}")
    if num_samples < 1:
        raise ValueError(f"num_samples must be >= 1, got {num_samples}")
    dev = device()
    pack = netpack(net, color_graph(moralize(net)))
    n = net.num_vars
    t_vars = np.asarray([t[0] for t in targets], dtype=np.int64)
    t_cases = np.asarray([t[1] for t in targets], dtype=np.int64)
    cases = context.num_cases
    db = DeviceBatch(n, 1, cases, cases, dev)
    dense = context.to_dense()
    db.set_latent_hint((dense < 0).mean() if dense.size else 0.0)
    obs = torch.full((n, db.pitch), -1, dtype=torch.int8, device=dev)
    if dense.size and dense.max() >= max(net.cardinalities):
        raise ValidationError("context contains a state >= its variable's cardinality")
    obs[:, :cases] = torch.from_numpy(dense.astype(np.int8)).to(dev)
    db.set_obs(obs)
    db.compute_ranks()
    s = stream_handle()
    err = ErrorWord(dev)

    rej = torch.empty(n * (_lib.REJ_SLACK + 2), dtype=torch.int64, device=dev)
    keys = var_keys(None, seed, "latent_init", (0,), n)
    _lib.call("sg_init_states", pack.ref, db.ref, obs.data_ptr(), db.pitch, _lib.SG_RNG_NUMPY, 0,
              keys.data_ptr(), rej.data_ptr(), err.ptr, s)
    _lib.call("sg_check_range", pack.ref, obs.data_ptr(), db.pitch, cases, err.ptr, s)
    cpt = torch.from_numpy(pack.flatten(cpts.tables)).to(dev)
    ptab = torch.empty(max(1, pack.layout.scalars["ptab_size"]), dtype=torch.float64, device=dev)
    ftab = torch.empty(pack.layout.scalars["ftab_size"] + 1, dtype=torch.int32, device=dev)
    _lib.call("sg_build_tables", pack.ref, cpt.data_ptr(), ptab.data_ptr(), ftab.data_ptr(), s)
    max_card = int(max((net.cardinalities[v] for v in t_vars), default=0))
    width = max(max_card, 1)
    freq = torch.zeros((len(t_vars), width), dtype=torch.int64, device=dev)
    tv = torch.from_numpy(t_vars.astype(np.int32)).to(dev)
    tc = torch.from_numpy(t_cases.astype(np.int32)).to(dev)
    for it in range(burn_in + num_samples):
        var_keys(keys, derive_seed(seed, "predict", it), "var", (), n)
        _lib.call("sg_sweep", pack.ref, db.ref, cpt.data_ptr(), ptab.data_ptr(), ftab.data_ptr(),
                  _lib.SG_RNG_NUMPY, 0, None, keys.data_ptr(), None, None, None, err.ptr, s)
        if it >= burn_in and len(t_vars):
            _lib.call("sg_predict_tally", db.states.data_ptr(), db.m * db.pitch, tv.data_ptr(), tc.data_ptr(),
                      len(t_vars), width, freq.data_ptr(), err.ptr, s)
    _raise_errors(err.read())
    if not len(t_vars):
        return np.zeros((0, 0))
    return freq.cpu().numpy()[:, :max_card].astype(np.float64) / num_samples

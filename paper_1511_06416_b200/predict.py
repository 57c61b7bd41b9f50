"""Held-out prediction with frozen CPTs (reference ``metrics.predict_missing``,
metrics.py:89-139), on the device.

The context's present entries stay clamped; every other cell is latent and is
resampled by ``burn_in + num_samples`` sweeps keyed ``derive_seed(seed,
"predict", it)`` (numpy RNG mode, so the result is bit-identical to the
reference).  The latent init is ``(seed, "latent_init", 0)`` as in the
reference.  Target states are gathered on the device after each kept sweep.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .device import ErrorWord, device, netpack, stream_handle
from .errors import DimensionMismatch
from .network import color_graph, moralize
from .rng import derive_seed, stream_key_ints
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
    obs[:, :cases] = torch.from_numpy(dense.astype(np.int8)).to(dev)
    db.set_obs(obs)
    db.compute_ranks()
    s = stream_handle()
    err = ErrorWord(dev)

    def keys_for(sd, label, *ctx):
        k = np.empty((n, 2), dtype=np.uint64)
        for v in range(n):
            k[v] = stream_key_ints(sd, label, *ctx, v)
        return torch.from_numpy(k.view(np.int64)).to(dev)

    rej = torch.empty(n * (_lib.REJ_SLACK + 2), dtype=torch.int64, device=dev)
    ikeys = keys_for(seed, "latent_init", 0)
    _lib.call("sg_init_states", pack.ref, db.ref, obs.data_ptr(), db.pitch, _lib.SG_RNG_NUMPY, 0,
              ikeys.data_ptr(), rej.data_ptr(), err.ptr, s)
    cpt = torch.from_numpy(pack.flatten(cpts.tables)).to(dev)
    ptab = torch.empty(max(1, pack.layout.scalars["ptab_size"]), dtype=torch.float64, device=dev)
    ftab = torch.empty(pack.layout.scalars["ftab_size"] + 1, dtype=torch.int32, device=dev)
    _lib.call("sg_build_tables", pack.ref, cpt.data_ptr(), ptab.data_ptr(), ftab.data_ptr(), s)
    max_card = int(max((net.cardinalities[v] for v in t_vars), default=0))
    freq = torch.zeros((len(t_vars), max(max_card, 1)), dtype=torch.float64, device=dev)
    tv = torch.from_numpy(t_vars).to(dev)
    tc = torch.from_numpy(t_cases).to(dev)
    rows = torch.arange(len(t_vars), device=dev)
    for it in range(burn_in + num_samples):
        keys = keys_for(derive_seed(seed, "predict", it), "var")
        _lib.call("sg_sweep", pack.ref, db.ref, cpt.data_ptr(), ptab.data_ptr(), ftab.data_ptr(),
                  _lib.SG_RNG_NUMPY, 0, None, keys.data_ptr(), None, None, None, err.ptr, s)
        if it >= burn_in and len(t_vars):
            states = (db.states[tv, 0, tc].to(torch.int64) & 0x7F)
            freq.index_put_((rows, states), torch.ones_like(rows, dtype=torch.float64), accumulate=True)
    _raise_errors(err.read())
    return (freq / num_samples).cpu().numpy()[:, :max_card] if len(t_vars) else np.zeros((0, 0))

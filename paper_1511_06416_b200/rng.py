"""Keyed counter-based random streams.

Every sampling site draws from its own Philox stream whose 128-bit key is the
blake2b-128 digest of ``"seed:label:i0:i1..."`` read as two little-endian
uint64 words (reference ``samegibbs/rng.py:16-30``).  The CUDA kernels consume
those keys directly:

* ``numpy`` RNG mode reproduces numpy's ``Philox4x64-10`` stream for a key
  word for word (``u_i = (philox(ctr=i//4+1, key)[i%4] >> 11) * 2**-53``),
  so a GPU sweep is bit-identical to the reference sweep;
* ``fast`` mode uses ``Philox4x32-10`` keyed by ``derive_seed`` of the same
  site with counters tied to (case, variable, replica quad), so results are
  independent of tiling and of how cases are sharded over GPUs.

Host-side hashing is a handful of calls per minibatch step; it is not on the
device path.
"""

from __future__ import annotations

import hashlib

import numpy as np


def _site_text(seed: int, label: str, indices) -> bytes:
    parts = [str(int(seed)), label]
    parts.extend(str(int(i)) for i in indices)
    return ":".join(parts).encode()


def stream_key(seed: int, label: str, *indices: int) -> np.ndarray:
    """128-bit Philox key of a sampling site, as ``uint64[2]``."""
    digest = hashlib.blake2b(_site_text(seed, label, indices), digest_size=16).digest()
    return np.array([int.from_bytes(digest[:8], "little"),
                     int.from_bytes(digest[8:], "little")], dtype=np.uint64)


def stream_key_ints(seed: int, label: str, *indices: int) -> tuple[int, int]:
    """Same key as :func:`stream_key`, as two Python ints (no numpy boxing)."""
    digest = hashlib.blake2b(_site_text(seed, label, indices), digest_size=16).digest()
    return int.from_bytes(digest[:8], "little"), int.from_bytes(digest[8:], "little")


def derive_seed(seed: int, label: str, *indices: int) -> int:
    """First key word of a site, used as a plain integer sub-seed."""
    return stream_key_ints(seed, label, *indices)[0]


def substream(seed: int, label: str, *indices: int) -> np.random.Generator:
    """numpy generator of a site (API compatibility; the device path never calls it)."""
    return np.random.Generator(np.random.Philox(key=stream_key(seed, label, *indices)))

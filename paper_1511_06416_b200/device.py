"""Device plumbing: the CUDA device, the current stream, cached network packs.

PyTorch is used only for device memory, streams and pinned host buffers; all
compute goes through the C-ABI library (``_lib``).  There is no CPU path: if
CUDA is unavailable every entry point raises :class:`DeviceError`.
"""

from __future__ import annotations

import threading

import torch

from . import _lib
from .errors import DeviceError
from .network import Coloring, Network


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: this backend runs only on a GPU (sm_100a)")
    _lib.load()
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


_pack_cache: dict = {}
_pack_lock = threading.Lock()


def netpack(net: Network, coloring: Coloring | None = None):
    """Cached :class:`NetPack` for a network (keyed by structure + colouring)."""
    from .netpack import NetPack

    dev = device()
    key = (net.cardinalities, net.parents, None if coloring is None else coloring.groups, dev.index)
    with _pack_lock:
        pack = _pack_cache.get(key)
        if pack is None:
            pack = NetPack(net, dev, coloring)
            if len(_pack_cache) > 64:
                _pack_cache.clear()
            _pack_cache[key] = pack
    return pack


class ErrorWord:
    """Device int32 error word with a pinned host mirror."""

    def __init__(self, dev: torch.device):
        self.dev = torch.zeros(1, dtype=torch.int32, device=dev)
        self.host = torch.zeros(1, dtype=torch.int32, pin_memory=True)

    @property
    def ptr(self) -> int:
        return self.dev.data_ptr()

    def reset(self) -> None:
        self.dev.zero_()

    def read(self) -> int:
        """Synchronising read of the accumulated flags."""
        self.host.copy_(self.dev, non_blocking=False)
        return int(self.host.item())



def site_keys(out: torch.Tensor, prefix: str, count: int, seed_dev: torch.Tensor | int | None = None,
              first: int = 0) -> torch.Tensor:
    """Device ``stream_key`` of ``count`` consecutive sites into ``out`` (int64 [count, 2]).

    Site i's text is ``[str(*seed_dev)] + prefix + str(first + i)`` (rng.py:16-20):
    ``site_keys(k, ":var:", n, seed_dev=cursor)`` = ``stream_key(seed, "var", v)``
    for v < n with the seed word read from device memory at replay time;
    ``site_keys(k, f"{seed}:latent_init:{p}:{mb}:", n)`` has the seed in the text.
    ``seed_dev`` is a device tensor (its first uint64) or a raw device pointer."""
    text = prefix.encode()
    ptr = None if seed_dev is None else (seed_dev if isinstance(seed_dev, int) else seed_dev.data_ptr())
    _lib.call("sg_site_keys", ptr, text, len(text), first, count, out.data_ptr(), stream_handle())
    return out


def var_keys(out: torch.Tensor | None, seed: int, label: str, context: tuple, n: int) -> torch.Tensor:
    """``stream_key(seed, label, *context, v)`` for v < n on the device (int64 [n, 2]).

    Hashed by ``sg_site_keys`` (one thread per variable); a site text that does
    not fit one BLAKE2b block (seeds beyond 64 bits) is hashed on the host."""
    if out is None:
        out = torch.empty((max(1, n), 2), dtype=torch.int64, device=device())
    prefix = ":".join([str(int(seed)), label, *(str(int(i)) for i in context)]) + ":"
    if len(prefix) <= 88:
        return site_keys(out, prefix, n)
    import numpy as np

    from .rng import stream_key_ints

    host = np.empty((n, 2), dtype=np.uint64)
    for v in range(n):
        host[v] = stream_key_ints(seed, label, *context, v)
    out[:n].copy_(torch.from_numpy(host.view(np.int64)))
    return out

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


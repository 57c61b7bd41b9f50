"""The C-ABI library builds, loads without a GPU and exports every entry point
that include/samegibbs_b200.h declares (no compute calls here)."""

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "samegibbs_b200.h"


def declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(sg_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_abi():
    names = declared()
    assert "sg_sweep" in names and "sg_build_tables" in names and len(names) >= 14


def test_library_exports_every_declared_symbol():
    from paper_1511_06416_b200 import _build, _lib

    _build.build()
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    for name in declared():
        assert hasattr(lib, name), name
    assert lib.sg_abi_version() == _lib.ABI_VERSION == 2
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    for name in declared():
        assert re.search(rf"\bT {name}\b", out), name


def test_python_binding_covers_the_header():
    from paper_1511_06416_b200 import _lib

    assert sorted(_lib.EXPORTED) == declared()


def test_struct_layout_matches_header():
    """ctypes mirrors of sg_net / sg_batch have the C layout (offsets checked by a tiny C probe)."""
    from paper_1511_06416_b200 import _lib

    probe = r'''
#include <stdio.h>
#include <stddef.h>
#include "samegibbs_b200.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(sg_net), offsetof(sg_net, cells),
         offsetof(sg_net, row_var), offsetof(sg_net, tally_chunk), sizeof(sg_batch), offsetof(sg_batch, case_base),
         offsetof(sg_batch, nmiss), sizeof(sg_finish), offsetof(sg_finish, flags), sizeof(sg_small));
  return 0;
}
'''
    import tempfile

    with tempfile.TemporaryDirectory() as td:
        src = Path(td) / "p.c"
        src.write_text(probe)
        exe = Path(td) / "p"
        subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
        got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    want = [ctypes.sizeof(_lib.SgNet), _lib.SgNet.cells.offset, _lib.SgNet.row_var.offset,
            _lib.SgNet.tally_chunk.offset, ctypes.sizeof(_lib.SgBatch), _lib.SgBatch.case_base.offset,
            _lib.SgBatch.nmiss.offset, ctypes.sizeof(_lib.SgFinish), _lib.SgFinish.flags.offset,
            ctypes.sizeof(_lib.SgSmall)]
    assert got == want


def test_no_cpu_fallback_without_gpu():
    """Without a CUDA device the product path refuses to run (no silent fallback)."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_1511_06416_b200 as sg
    from paper_1511_06416_b200.errors import DeviceError

    net = sg.build_network([2, 2], [(0, 1)])
    with pytest.raises(DeviceError):
        sg.tally_counts(net, [[0, 1], [1, 1]], [1.0, 1.0])


def test_device_site_key_hash_matches_hashlib():
    """sg_site_keys' BLAKE2b-128 (evaluated on the host through sg_site_key_host,
    the same __host__ __device__ code) equals rng.stream_key (hashlib), rng.py:16-20."""
    import hashlib

    import numpy as np

    from paper_1511_06416_b200 import _build, _lib
    from paper_1511_06416_b200.rng import stream_key_ints

    _build.build()
    lib = _lib.load()
    texts = [b"", b"a", b"0:sweep:0:0:0", b"18446744073709551615:var:999", b"-7:latent_init:3:1:2",
             b"x" * 127, b"y" * 128, b"300:cpt_update:1:2"]
    out = (ctypes.c_uint64 * 2)()
    for t in texts:
        assert lib.sg_site_key_host(t, len(t), out) == 0
        d = hashlib.blake2b(t, digest_size=16).digest()
        assert (out[0], out[1]) == (int.from_bytes(d[:8], "little"), int.from_bytes(d[8:], "little")), t
    rng = np.random.default_rng(0)
    for _ in range(200):
        seed = int(rng.integers(0, 2**63)) * int(rng.integers(1, 3))
        v = int(rng.integers(0, 10**6))
        t = f"{seed}:var:{v}".encode()
        assert lib.sg_site_key_host(t, len(t), out) == 0
        assert (out[0], out[1]) == stream_key_ints(seed, "var", v)

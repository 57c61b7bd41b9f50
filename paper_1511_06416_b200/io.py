"""Network / CPT JSON files (reference ``samegibbs/io.py:53-102``) and the
binary ``.sgb`` observation format with its streaming source.

A network file is a JSON object with ``cardinalities``, ``edges`` (list of
[parent, child]) and optional ``cpts`` (one row-major list per variable, rows
indexed by the ascending-parent mixed radix).  A CPT checkpoint is the same
schema with ``cpts`` present.
"""

from __future__ import annotations

import json
import struct
from pathlib import Path

import numpy as np
import torch

from .datagen import _BlockStream
from .errors import IoError, ParseError
from .model import CptSet
from .network import Network, build_network

_DATA = Path(__file__).resolve().parent / "data"


def bundled_network_path(name: str) -> Path:
    p = _DATA / f"{name}.json"
    if not p.is_file():
        raise IoError(f"no bundled network named {name!r}")
    return p


def load_network_file(path) -> tuple[Network, CptSet | None]:
    p = Path(path)
    if not p.exists():
        raise IoError(f"file not found: {p}")
    try:
        obj = json.loads(p.read_text())
    except json.JSONDecodeError as exc:
        raise ParseError(f"{p}:{exc.lineno}: {exc.msg}") from exc
    for key in ("cardinalities", "edges"):
        if key not in obj:
            raise ParseError(f"{p}: missing required field {key!r}")
    try:
        net = build_network([int(c) for c in obj["cardinalities"]], [(int(a), int(b)) for a, b in obj["edges"]])
    except (TypeError, ValueError) as exc:
        raise ParseError(f"{p}: malformed network fields: {exc}") from exc
    raw = obj.get("cpts")
    if raw is None:
        return net, None
    if len(raw) != net.num_vars:
        raise ParseError(f"{p}: cpts has {len(raw)} tables for {net.num_vars} variables")
    tables = []
    for v, flat in enumerate(raw):
        rows, card = net.table_shape(v)
        a = np.asarray(flat, dtype=np.float64)
        if a.size != rows * card:
            raise ParseError(f"{p}: cpts[{v}] has {a.size} entries, expected {rows * card}")
        tables.append(a.reshape(rows, card))
    cpts = CptSet(tables)
    try:
        cpts.validate()
    except ValueError as exc:
        raise ParseError(f"{p}: {exc}") from exc
    return net, cpts


def write_network_file(path, net: Network, cpts: CptSet | None = None) -> None:
    obj: dict = {"cardinalities": list(net.cardinalities),
                 "edges": sorted([p, c] for c in range(net.num_vars) for p in net.parents[c])}
    if cpts is not None:
        obj["cpts"] = [np.asarray(t).ravel().tolist() for t in cpts.tables]
    Path(path).write_text(json.dumps(obj, indent=1) + "\n")


# ---------------------------------------------------------------- binary observation files
#
# The reference's data files are text (io.py:105-153: CSV triples read through
# pandas), which cannot feed a GPU at 10^8 cases x 1000 variables.  ``.sgb``
# stores the observation matrix in the layout the device consumes, as
# minibatch blocks:
#
#   header (64 bytes, little endian): b"SGB1", version u32 = 1, num_vars u32,
#       num_cases u64, block_cases u32, pitch u32, encoding u32 (0 = int8,
#       1 = 4-bit), zero padding
#   blocks: ceil(num_cases / block_cases) x num_vars rows of `pitch` cases
#       (case c of block b = case b * block_cases + c; columns past the data
#       are missing).  int8: one byte per cell, -1 = missing.  4-bit: two
#       cells per byte (case 2j in the low nibble), 15 = missing, so cards
#       <= 15; decoded on the device by sg_unpack_nibbles.  2-bit ("crumb",
#       encoding 2): four cells per byte (case 4j + h in bits 2h..2h+1), 3 =
#       missing, cards <= 3; decoded by sg_unpack_crumbs.

_SGB_MAGIC = b"SGB1"
_SGB_ENCODINGS = {"int8": 0, "nibble": 1, "crumb": 2}
_SGB_HEADER = struct.Struct("<4sIIQIII")


def pack_bits(block, pitch: int, bits: int):
    """(n, cases) observation block (int, -1 = missing) -> the packed .sgb
    form with ``bits`` = 4 or 2 bits per cell: uint8 (n, pitch * bits / 8),
    case k * (8 / bits) + h in bits [h * bits, (h + 1) * bits) of byte k, the
    all-ones value = missing (also for the padding columns up to ``pitch``, a
    multiple of 64).  Works on numpy arrays and on (host or device) tensors."""
    if bits not in (4, 2):
        raise ValueError("bits must be 4 or 2")
    per = 8 // bits
    miss = (1 << bits) - 1
    if pitch % 64 or pitch < block.shape[1]:
        raise ValueError("pitch must be a multiple of 64 covering the block")
    if isinstance(block, torch.Tensor):
        u = torch.full((block.shape[0], pitch), miss, dtype=torch.uint8, device=block.device)
        b = block.to(torch.int16)
        u[:, :block.shape[1]] = torch.where(b < 0, miss, b).to(torch.uint8)
        out = u[:, 0::per].clone()
        for h in range(1, per):
            out |= u[:, h::per] << (bits * h)
        return out
    arr = np.asarray(block)
    u = np.full((arr.shape[0], pitch), miss, dtype=np.uint8)
    u[:, :arr.shape[1]] = np.where(arr < 0, miss, arr).astype(np.uint8)
    out = u[:, 0::per].copy()
    for h in range(1, per):
        out |= (u[:, h::per] << (bits * h)).astype(np.uint8)
    return out


def pack_nibbles(block, pitch: int):
    """The 4-bit .sgb form (:func:`pack_bits` with bits = 4)."""
    return pack_bits(block, pitch, 4)


def pack_crumbs(block, pitch: int):
    """The 2-bit .sgb form (:func:`pack_bits` with bits = 2; cards <= 3)."""
    return pack_bits(block, pitch, 2)


def write_binary(path, data, block_cases: int, encoding: str = "int8") -> None:
    """Write a DataMatrix or a dense (num_vars, num_cases) int matrix (-1 = missing) as ``.sgb``."""
    from .datagen import DataMatrix

    if encoding not in _SGB_ENCODINGS:
        raise ValueError(f"encoding must be one of {tuple(_SGB_ENCODINGS)}, got {encoding!r}")
    if isinstance(data, DataMatrix):
        dense = data.to_dense()
    else:
        dense = np.asarray(data.cpu() if hasattr(data, "cpu") else data)
    n, cases = dense.shape
    if cases == 0:
        raise ValueError("no cases to write")
    limit = {"int8": 128, "nibble": 15, "crumb": 3}[encoding]
    if dense.max(initial=-1) >= limit or dense.min(initial=0) < -1:
        raise ValueError(f"states must lie in [-1, {limit - 1}] for the {encoding} encoding")
    pitch = max(64, (block_cases + 63) // 64 * 64)
    nb = (cases + block_cases - 1) // block_cases
    with open(path, "wb") as f:
        head = _SGB_HEADER.pack(_SGB_MAGIC, 1, n, cases, block_cases, pitch, _SGB_ENCODINGS[encoding])
        f.write(head + bytes(64 - len(head)))
        for b in range(nb):
            lo, hi = b * block_cases, min(cases, (b + 1) * block_cases)
            blk = np.full((n, pitch), -1, dtype=np.int8)
            blk[:, :hi - lo] = dense[:, lo:hi]
            if encoding != "int8":
                blk = pack_bits(blk, pitch, 4 if encoding == "nibble" else 2)
            f.write(blk.tobytes())


def write_binary_blocks(path, num_vars: int, num_cases: int, block_cases: int, block_fn,
                        encoding: str = "nibble") -> None:
    """Stream an ``.sgb`` file block by block: ``block_fn(lo, hi)`` returns the
    (num_vars, hi - lo) observations of cases [lo, hi) (-1 = missing; a host
    array or a device tensor, packed on its own device).  Lets a generator
    write files far larger than host memory (BASELINE C5)."""
    import torch

    if encoding not in _SGB_ENCODINGS:
        raise ValueError(f"encoding must be one of {tuple(_SGB_ENCODINGS)}, got {encoding!r}")
    if num_cases <= 0:
        raise ValueError("no cases to write")
    limit = {"int8": 128, "nibble": 15, "crumb": 3}[encoding]
    pitch = max(64, (block_cases + 63) // 64 * 64)
    nb = (num_cases + block_cases - 1) // block_cases
    with open(path, "wb") as f:
        head = _SGB_HEADER.pack(_SGB_MAGIC, 1, num_vars, num_cases, block_cases, pitch, _SGB_ENCODINGS[encoding])
        f.write(head + bytes(64 - len(head)))
        for b in range(nb):
            lo, hi = b * block_cases, min(num_cases, (b + 1) * block_cases)
            blk = block_fn(lo, hi)
            if tuple(blk.shape) != (num_vars, hi - lo):
                raise ValueError(f"block {b}: expected shape {(num_vars, hi - lo)}, got {tuple(blk.shape)}")
            if isinstance(blk, torch.Tensor):
                if int(blk.max()) >= limit or int(blk.min()) < -1:
                    raise ValueError(f"states must lie in [-1, {limit - 1}] for the {encoding} encoding")
                if encoding == "int8":
                    out = torch.full((num_vars, pitch), -1, dtype=torch.int8, device=blk.device)
                    out[:, :hi - lo] = blk
                else:
                    out = pack_bits(blk, pitch, 4 if encoding == "nibble" else 2)
                f.write(out.cpu().numpy().tobytes())
            else:
                arr = np.asarray(blk)
                if arr.max(initial=-1) >= limit or arr.min(initial=0) < -1:
                    raise ValueError(f"states must lie in [-1, {limit - 1}] for the {encoding} encoding")
                out = np.full((num_vars, pitch), -1, dtype=np.int8)
                out[:, :hi - lo] = arr
                if encoding != "int8":
                    out = pack_bits(out, pitch, 4 if encoding == "nibble" else 2)
                f.write(out.tobytes())


def read_binary_header(path) -> dict:
    with open(path, "rb") as f:
        raw = f.read(64)
    if len(raw) < 64:
        raise IoError(f"{path}: truncated header")
    magic, version, n, cases, block, pitch, enc = _SGB_HEADER.unpack(raw[:_SGB_HEADER.size])
    names = {v: k for k, v in _SGB_ENCODINGS.items()}
    if magic != _SGB_MAGIC or version != 1 or enc not in names:
        raise ParseError(f"{path}: not an .sgb v1 file")
    return {"num_vars": n, "num_cases": cases, "block_cases": block, "pitch": pitch, "encoding": names[enc]}


class BinaryFileSource(_BlockStream):
    """Minibatch source streaming an ``.sgb`` file from disk (reference source
    protocol, sampler.py:393-398; ``FileSource`` io.py:156-240 for text).

    Minibatches are the file's blocks.  Block i+1 is read from disk straight
    into one of two pinned buffers and copied on a side stream while the
    consumer works on block i (4-bit files are decoded on the device).
    ``cycle`` replays the file that many times per pass.
    """

    def __init__(self, path, cycle: int = 1):
        h = read_binary_header(path)
        self.path = Path(path)
        self.header = h
        self.bits = {"int8": 8, "nibble": 4, "crumb": 2}[h["encoding"]]
        self._row_bytes = h["pitch"] * self.bits // 8
        self._block_bytes = h["num_vars"] * self._row_bytes
        self._nb = (h["num_cases"] + h["block_cases"] - 1) // h["block_cases"]
        size = self.path.stat().st_size
        if size < 64 + self._nb * self._block_bytes:
            raise IoError(f"{path}: truncated ({size} bytes)")
        self._setup(h["num_vars"], h["pitch"], h["num_cases"], h["block_cases"], cycle)
        dt = torch.uint8 if self.bits < 8 else torch.int8
        self._pinned = [torch.empty((h["num_vars"], self._row_bytes), dtype=dt).pin_memory() for _ in range(2)]
        self._pinned_ev = [None, None]
        self._turn = 0
        self._pending = 0
        self._file = None

    def _num_blocks(self) -> int:
        return self._nb

    def _host_block(self, i: int) -> torch.Tensor:
        k = self._turn
        self._turn ^= 1
        if self._pinned_ev[k] is not None:
            self._pinned_ev[k].synchronize()  # the previous copy out of this buffer has drained
        if self._file is None:
            self._file = open(self.path, "rb", buffering=0)
        self._file.seek(64 + i * self._block_bytes)
        got = self._file.readinto(memoryview(self._pinned[k].numpy()).cast("B"))
        if got != self._block_bytes:
            raise IoError(f"{self.path}: short read of block {i}")
        self._pending = k
        return self._pinned[k]

    def _copy(self, i: int, slot: int, after):
        ev = super()._copy(i, slot, after)
        self._pinned_ev[self._pending] = ev
        return ev


# ------------------------------------------------------------------ text formats of the reference CLI
# (io.py:105-153 coordinate data, io.py:243-270 trace CSV, io.py:273-280 manifest):
# read so that `train` can consume the reference's own files.

def write_data(path, data) -> None:
    """Coordinate triples, case-major, 1-based (reference io.py:105-116)."""
    with open(path, "w") as fh:
        fh.write(f"{data.num_vars} {data.num_cases} {data.nnz}\n")
        trip = np.stack([data.var_idx + 1, data.case_idx + 1, data.values.astype(np.int64) + 1], axis=1)
        np.savetxt(fh, trip, fmt="%d", delimiter=" ")


def read_data(path):
    """A whole coordinate file as a DataMatrix (reference io.py:119-153)."""
    from .datagen import DataMatrix

    path = Path(path)
    if not path.exists():
        raise IoError(f"file not found: {path}")
    with open(path) as fh:
        header = fh.readline()
        try:
            num_vars, num_cases, nnz = (int(tok) for tok in header.split())
        except ValueError as exc:
            raise ParseError(f"{path}:1: bad header {header.strip()!r}") from exc
        body = fh.read()
    try:
        trip = np.array(body.split(), dtype=np.int64).reshape(-1, 3) if body.strip() else np.zeros((0, 3), np.int64)
    except ValueError as exc:
        raise ParseError(f"{path}: bad triple row: {exc}") from exc
    if len(trip) != nnz:
        raise ParseError(f"{path}: header promises {nnz} entries, found {len(trip)}")
    try:
        return DataMatrix(num_vars=num_vars, num_cases=num_cases, var_idx=trip[:, 0] - 1, case_idx=trip[:, 1] - 1,
                          values=trip[:, 2] - 1)
    except ValueError as exc:
        raise ParseError(f"{path}: {exc}") from exc


def write_trace(path, trace) -> None:
    """pass,seconds,kl_avg,vars_per_sec rows (reference io.py:243-249)."""
    with open(path, "w") as fh:
        fh.write("pass,seconds,kl_avg,vars_per_sec\n")
        for r in trace.records:
            kl = "" if r.kl_avg is None else repr(r.kl_avg)
            vps = "" if r.vars_per_sec is None else repr(r.vars_per_sec)
            fh.write(f"{r.pass_index},{r.seconds!r},{kl},{vps}\n")


def read_trace(path):
    from .sampler import Trace, TraceRecord

    trace = Trace()
    with open(path) as fh:
        if fh.readline().strip() != "pass,seconds,kl_avg,vars_per_sec":
            raise ParseError(f"{path}:1: unexpected trace header")
        for line in fh:
            pass_ix, seconds, kl, vps = line.rstrip("\n").split(",")
            trace.records.append(TraceRecord(pass_index=int(pass_ix), seconds=float(seconds),
                                             kl_avg=float(kl) if kl else None,
                                             vars_per_sec=float(vps) if vps else None, vars_sampled=0))
    return trace


def write_manifest(path, manifest: dict) -> None:
    with open(path, "w") as fh:
        json.dump(manifest, fh, indent=1, sort_keys=True)
        fh.write("\n")


def read_manifest(path) -> dict:
    try:
        with open(path) as fh:
            return json.load(fh)
    except FileNotFoundError as exc:
        raise IoError(f"file not found: {path}") from exc
    except json.JSONDecodeError as exc:
        raise ParseError(f"{path}: {exc}") from exc

"""Network / CPT JSON files (reference ``samegibbs/io.py:53-102``).

A network file is a JSON object with ``cardinalities``, ``edges`` (list of
[parent, child]) and optional ``cpts`` (one row-major list per variable, rows
indexed by the ascending-parent mixed radix).  A CPT checkpoint is the same
schema with ``cpts`` present.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

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

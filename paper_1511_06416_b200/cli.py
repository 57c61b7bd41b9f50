"""Command-line backend of ``samegibbs train`` on the device.

Mirrors the reference's ``cmd_train`` (cli.py:112-165): the same flags, the
same outputs (``cpts.json``, ``trace.csv``, ``manifest.json``), the same exit
codes (0 success, 2 validation / parse error, 3 runtime error), and
``--from-manifest`` replay.  What changes is the backend: the run goes
through this package's ``run()`` (CUDA kernels, no CPU path) and the data
may be the reference's coordinate text file or an ``.sgb`` binary file
(streamed from disk by :class:`~paper_1511_06416_b200.io.BinaryFileSource`).
``convert`` writes an ``.sgb`` file from a coordinate file.

    python -m paper_1511_06416_b200 train --backend cuda --network koller --data d.mm --out out/ ...
    python -m paper_1511_06416_b200 convert --data d.mm --out d.sgb --block-cases 12500 [--encoding nibble]

The reference-side switch (``samegibbs train --backend cuda`` delegating here)
is shown in INTEGRATION.md.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

from . import io
from .errors import ParseError, SamGibbsError, ValidationError
from .metrics import throughput
from .model import DirichletPrior
from .sampler import RNG_MODES, SamplerConfig, run

BACKENDS = ("cuda",)


def _network_path(spec: str) -> Path:
    """A plain path, or the name of a bundled network like ``koller`` (cli.py:27-33)."""
    path = Path(spec)
    if not path.exists() and "/" not in spec and not spec.endswith(".json"):
        return io.bundled_network_path(spec)
    return path


def _parse_schedule(text: str) -> tuple[tuple[int, int], ...]:
    """``1x50,5x150`` -> ((1, 50), (5, 150)) (cli.py:36-45)."""
    pieces = []
    for piece in text.split(","):
        try:
            m, passes = piece.strip().split("x")
            pieces.append((int(m), int(passes)))
        except ValueError as exc:
            raise ValidationError(f"bad schedule piece {piece!r}, expected MxPASSES") from exc
    return tuple(pieces)


MANIFEST_KEYS = ("network", "data", "truth", "same_m", "same_schedule", "minibatch_size", "passes", "alpha",
                 "accumulator", "exp_decay", "sweeps_per_minibatch", "map_estimate", "seed", "threads")


def _manifest(args: argparse.Namespace) -> dict:
    out = {"command": "train", "backend": args.backend, "rng": args.rng}
    for key in MANIFEST_KEYS:
        val = getattr(args, key)
        out[key] = str(val) if key in ("network", "data") else (str(val) if key == "truth" and val else val)
    return out


def _apply_manifest(args: argparse.Namespace) -> None:
    manifest = io.read_manifest(args.from_manifest)
    if manifest.get("command") != "train":
        raise ParseError(f"{args.from_manifest}: not a train manifest")
    for key in MANIFEST_KEYS:
        if key not in manifest:
            raise ParseError(f"{args.from_manifest}: manifest missing field {key!r}")
        setattr(args, key, manifest[key])
    for key in ("backend", "rng"):
        if key in manifest:
            setattr(args, key, manifest[key])
    if args.same_schedule is not None and not isinstance(args.same_schedule, str):
        args.same_schedule = ",".join(f"{m}x{p}" for m, p in args.same_schedule)


def _source(path: str, minibatch_size: int):
    """An .sgb file streams from disk (its block size must equal the minibatch
    size); a coordinate text file is read whole (the reference's FileSource
    streams it; here it becomes an in-memory DataMatrix)."""
    p = Path(path)
    if not p.exists():
        raise ValidationError(f"data file not found: {p}")
    with open(p, "rb") as fh:
        magic = fh.read(4)
    if magic == io._SGB_MAGIC:
        src = io.BinaryFileSource(p)
        if src.minibatch_size != minibatch_size:
            raise ValidationError(f"{p}: .sgb blocks hold {src.minibatch_size} cases, --minibatch-size is "
                                  f"{minibatch_size} (convert with --block-cases {minibatch_size})")
        return src, src.num_cases
    data = io.read_data(p)
    return data, data.num_cases


def cmd_train(args: argparse.Namespace) -> int:
    if args.from_manifest:
        _apply_manifest(args)
    if args.backend not in BACKENDS:
        raise ValidationError(f"--backend must be one of {BACKENDS}")
    if args.network is None or args.data is None:
        raise ValidationError("train needs --network and --data (or --from-manifest)")
    net, _ = io.load_network_file(_network_path(args.network))
    truth = None
    if args.truth:
        truth_net, truth = io.load_network_file(_network_path(args.truth))
        if truth is None:
            raise ValidationError(f"{args.truth}: truth file has no cpts")
        if truth_net.cardinalities != net.cardinalities or truth_net.parents != net.parents:
            raise ValidationError("truth network structure differs from --network")
    if args.same_schedule and args.same_m != 1:
        raise ValidationError("give either --same-m or --same-schedule, not both")
    same_m = _parse_schedule(args.same_schedule) if args.same_schedule else args.same_m
    try:
        cfg = SamplerConfig(same_m=same_m, minibatch_size=args.minibatch_size, num_passes=args.passes,
                            prior=DirichletPrior(args.alpha),
                            accumulator_mode="moving_sum" if args.accumulator == "moving" else "exponential",
                            exp_decay=args.exp_decay, sweeps_per_minibatch=args.sweeps_per_minibatch,
                            map_estimate=args.map_estimate, seed=args.seed, rng=args.rng)
    except ValueError as exc:
        raise ValidationError(str(exc)) from exc
    source, num_cases = _source(args.data, cfg.minibatch_size)
    out_dir = Path(args.out)
    out_dir.mkdir(parents=True, exist_ok=True)
    started = time.perf_counter()
    cpts, trace = run(net, source, cfg, truth=truth, threads=args.threads)
    elapsed = time.perf_counter() - started
    io.write_network_file(out_dir / "cpts.json", net, cpts)
    io.write_trace(out_dir / "trace.csv", trace)
    io.write_manifest(out_dir / "manifest.json", _manifest(args))
    summary = {"elapsed_seconds": round(elapsed, 3), "passes": args.passes, "cases": num_cases,
               "backend": args.backend, "rng": args.rng}
    if trace.records:
        summary["vars_per_sec_overall"] = throughput(trace).overall
        if truth is not None:
            summary["final_kl_avg"] = trace.records[-1].kl_avg
    print(json.dumps(summary))
    print(f"wrote {out_dir / 'cpts.json'}, {out_dir / 'trace.csv'}, {out_dir / 'manifest.json'}")
    return 0


def cmd_convert(args: argparse.Namespace) -> int:
    data = io.read_data(args.data)
    io.write_binary(args.out, data, args.block_cases, args.encoding)
    print(f"wrote {args.out}: {data.num_vars} vars x {data.num_cases} cases, {args.encoding} blocks of "
          f"{args.block_cases} cases")
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_1511_06416_b200", description=__doc__.split("\n")[0])
    sub = ap.add_subparsers(dest="command", required=True)
    train = sub.add_parser("train", help="stream a data file and learn CPTs on the GPU")
    train.add_argument("--backend", choices=BACKENDS, default="cuda")
    train.add_argument("--network")
    train.add_argument("--data", help="coordinate text file (reference format) or .sgb binary file")
    train.add_argument("--out", required=True, help="output directory")
    train.add_argument("--truth", help="network+cpts file for KL tracing")
    train.add_argument("--same-m", type=int, default=1, dest="same_m")
    train.add_argument("--same-schedule", dest="same_schedule", help="annealing schedule, e.g. 1x50,5x150")
    train.add_argument("--minibatch-size", type=int, default=1024)
    train.add_argument("--passes", type=int, default=1)
    train.add_argument("--alpha", type=float, default=1.0)
    train.add_argument("--accumulator", choices=("moving", "exp"), default="moving")
    train.add_argument("--exp-decay", type=float, default=1.0)
    train.add_argument("--sweeps-per-minibatch", type=int, default=1)
    train.add_argument("--map-estimate", action="store_true")
    train.add_argument("--seed", type=int, default=0)
    train.add_argument("--threads", type=int, default=1, help="accepted for compatibility; never changes results")
    train.add_argument("--rng", choices=RNG_MODES, default="numpy",
                       help="numpy: the reference's own streams (bit-exact sweeps); fast / joint: device streams")
    train.add_argument("--from-manifest", help="replay a previous run's manifest")
    train.set_defaults(func=cmd_train)
    conv = sub.add_parser("convert", help="coordinate text file -> .sgb binary blocks")
    conv.add_argument("--data", required=True)
    conv.add_argument("--out", required=True)
    conv.add_argument("--block-cases", type=int, required=True)
    conv.add_argument("--encoding", choices=("int8", "nibble", "crumb"), default="nibble")
    conv.set_defaults(func=cmd_convert)
    return ap


def main(argv: list[str] | None = None) -> int:
    """Exit codes of the reference CLI (cli.py:1-6): 0 ok, 2 validation/parse, 3 runtime."""
    ap = build_parser()
    try:
        args = ap.parse_args(argv)
    except SystemExit as exc:
        return int(exc.code or 0)
    try:
        return args.func(args)
    except ValidationError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    except SamGibbsError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 3


if __name__ == "__main__":
    sys.exit(main())

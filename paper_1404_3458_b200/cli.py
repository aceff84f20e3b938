"""Command-line tool on the GPU codec (reference cli.py:1-142).

    python -m paper_1404_3458_b200.cli encode --in FILE --out DIR [--r 8|16] [--k K]
    python -m paper_1404_3458_b200.cli decode --shards DIR --out FILE

Same arguments, outputs and shard files as `binfec encode/decode`; the
stripe packing, encode and decode run on the GPU (shardfile.py here).  The
reference's `selftest` and `bench` subcommands are out of scope (the test
suite and bench.py cover them).
"""

from __future__ import annotations

import argparse
import sys

from .shardfile import decode_file, encode_bytes, _write_payloads


def _cmd_encode(args: argparse.Namespace) -> int:
    r, k = args.r, args.k
    if k < 1 or k & (k - 1) or k >= (1 << r):
        raise ValueError(f"k must be a power of two below {1 << r}, got {k}")
    with open(args.input, "rb") as fh:
        data = fh.read()
    header, payloads = encode_bytes(data, r, k)
    paths = _write_payloads(args.outdir, header, payloads)
    print(f"wrote {len(paths)} shards ({header.stripe_count} stripes, k={k}, n={header.n}) "
          f"to {args.outdir}")
    return 0


def _cmd_decode(args: argparse.Namespace) -> int:
    nbytes, used, skipped = decode_file(args.shards, args.output)
    for note in skipped:
        print(f"warning: skipping {note}", file=sys.stderr)
    print(f"reconstructed {nbytes} bytes from {used} shards to {args.output}")
    return 0


def main(argv: list[str] | None = None) -> int:
    parser = argparse.ArgumentParser(
        prog="binfec-b200",
        description="Erasure-code files into shards on the GPU; any k of n rebuild the original.")
    sub = parser.add_subparsers(dest="command", required=True)
    enc = sub.add_parser("encode", help="split a file into shards")
    enc.add_argument("--in", dest="input", required=True, metavar="FILE")
    enc.add_argument("--out", dest="outdir", required=True, metavar="DIR")
    enc.add_argument("--r", type=int, default=8, choices=(8, 16))
    enc.add_argument("--k", type=int, default=128)
    enc.set_defaults(func=_cmd_encode)
    dec = sub.add_parser("decode", help="rebuild a file from shards")
    dec.add_argument("--shards", required=True, metavar="DIR")
    dec.add_argument("--out", dest="output", required=True, metavar="FILE")
    dec.set_defaults(func=_cmd_decode)
    args = parser.parse_args(argv)
    return args.func(args)


if __name__ == "__main__":
    sys.exit(main())

"""`python -m paper_2508_14568_b200 compute|batch|table|eqcost ...` — the
reference CLI's subcommands (cli.cpp:240-330): compute and batch on the GPU
path, table (the product's own lookup tables) and eqcost (plaintext).

Same flags, LEUVEN_BUDGET default (cli.cpp:131-147), exit codes
(classify_error_exit, cli.cpp:121-129: 3 band too narrow, 2 input/params,
1 other) and report formats (print_human_report cli.cpp:110-119,
report_json cli.cpp:93-107). `--threads` is accepted for compatibility:
the batch is already traversed as one wavefront over all pairs.
"""
import argparse
import os
import sys

from . import BandTooNarrow, CharNotInAlphabet, CharNotInSubset, Error, FormatError
from . import InvalidParams, OutOfRangeValue
from . import leuven


def _env_budget() -> float:
    env = os.environ.get("LEUVEN_BUDGET", "")
    if not env:
        return 4000.0
    try:
        return float(env)
    except ValueError:
        raise InvalidParams(f"invalid LEUVEN_BUDGET value '{env}'")


def _exit_code(e: Error) -> int:
    if isinstance(e, BandTooNarrow):
        return 3
    if isinstance(e, (CharNotInAlphabet, CharNotInSubset, FormatError, InvalidParams,
                      OutOfRangeValue)):
        return 2
    return 1


def _human(r: dict) -> str:
    return (f"distance: {r['distance']}\n"
            f"mode: {r['mode']} (half-width {r['half_width']})\n"
            f"visited cells: {r['visited_cells']}\n"
            f"bootstraps: total {r['pbs_total']} (equality {r['pbs_equality']}, kernel "
            f"{r['pbs_kernel']}, refresh {r['refresh_count']}, preprocessing "
            f"{r['preprocessing_pbs']})\n"
            f"max key variance: {r['max_key_variance']} eps^2\n"
            f"wall time: {r['wall_time_ms']} ms\n")


def _flags(p):
    p.add_argument("--mode", default="exact", choices=["exact", "skip", "approx"])
    p.add_argument("--ell", type=int, default=None)
    p.add_argument("--encoding", default="ascii7")
    p.add_argument("--budget", type=float, default=None)
    p.add_argument("--key-encoding", default="negated", choices=["negated", "original"])
    p.add_argument("--preprocess", action="store_true")


def main(argv=None, out=sys.stdout, err=sys.stderr) -> int:
    ap = argparse.ArgumentParser(prog="leuven",
                                 description="encrypted edit distance with one bootstrap per cell")
    sub = ap.add_subparsers(dest="cmd", required=True)
    c = sub.add_parser("compute", help="distance of two strings")
    c.add_argument("--a", required=True)
    c.add_argument("--b", required=True)
    _flags(c)
    c.add_argument("--json", action="store_true")
    b = sub.add_parser("batch", help='JSONL of {"a":...,"b":...} pairs')
    b.add_argument("--input", required=True)
    b.add_argument("--threads", type=int, default=1)
    _flags(b)
    tb = sub.add_parser("table", help="dump a lookup table")
    tb.add_argument("which", help="minlut-original | minlut-negated | eqlut | eqlut9")
    ec = sub.add_parser("eqcost", help="equality bootstrap-cost table as CSV")
    ec.add_argument("--max-bits", type=int, default=16, choices=range(1, 65), metavar="[1-64]")
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 2
    if args.cmd == "table":  # cli.cpp:212-228
        if args.which not in ("minlut-original", "minlut-negated", "eqlut", "eqlut9"):
            err.write(f"unknown table '{args.which}'\n")
            return 2
        out.write(leuven.lut_dump(args.which))
        return 0
    if args.cmd == "eqcost":  # cli.cpp:230-238
        out.write("bits,standard,ours,combined\n")
        for bits in range(1, args.max_bits + 1):
            out.write(f"{bits},{leuven.eq_cost('standard_2bit', bits)},"
                      f"{leuven.eq_cost('ours_4bit', bits)},{leuven.eq_cost('combined', bits)}\n")
        return 0
    try:
        budget = args.budget if args.budget is not None else _env_budget()
        if args.cmd == "compute":
            rep = leuven.compute(args.a, args.b, args.mode, args.ell, args.encoding, budget,
                                 args.key_encoding, args.preprocess, include_timing=True)
            out.write(leuven.report_json(rep, include_timing=True) + "\n" if args.json
                      else _human(rep))
            return 0
        try:
            with open(args.input, encoding="utf-8") as fh:
                lines = fh.read().splitlines()
        except OSError:
            err.write(f"cannot open batch input: {args.input}\n")
            return 2
        for line in leuven.run_batch(lines, args.mode, args.ell, args.encoding, budget,
                                     args.key_encoding, args.preprocess):
            out.write(line + "\n")
        return 0
    except Error as e:
        err.write(f"{e}\n")
        return _exit_code(e)


if __name__ == "__main__":
    sys.exit(main())

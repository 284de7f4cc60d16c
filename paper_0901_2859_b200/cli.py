"""Command-line front end: batched tridiagonal solves from text files.

Mirrors the reference CLI's `solve` subcommand (tools/main.cpp:55-125,
options :277-289) on the GPU path:

    python -m paper_0901_2859_b200.cli [--workers W] [--verify] solve \
        --matrix M --rhs R [--partition b1,b2,...] [--out X] [--stats S]

* text formats of core/tridiag.hpp:158-212: the matrix file is the order
  n, then the sub, diag and super rows; the RHS file is a header `n N` and
  N rows of n values; blank lines are skipped; malformed input raises
  ParseError with the 1-based line number (tridiag.hpp:115-145);
* partition: `--partition` boundaries (Partition::parse,
  dichotomy/partition.hpp:52-72), else decompose(n, workers) when
  workers > 1, else no boundary (main.cpp:64-70);
* exit codes: 0 ok, 2 parse error, 3 solver error, 4 verification failure
  (main.cpp:23-25); `--verify` re-checks every solution against a banded
  dense-LU oracle at max-norm relative 1e-9 (main.cpp:92-111);
* the solutions are written as an RHS series with 17 significant digits
  (write_rhs_series, tridiag.hpp:187-196) and the run stats as the JSON of
  RunStats::to_json (runtime/run.hpp:42-51).
"""
from __future__ import annotations

import argparse
import json
import re
import sys
import time

import numpy as np

EXIT_PARSE, EXIT_SOLVER, EXIT_VERIFY = 2, 3, 4


class ParseError(ValueError):
    """core/errors.hpp:65-70: malformed text input with its 1-based line."""

    def __init__(self, line: int, msg: str):
        super().__init__(f"line {line}: {msg}")
        self.line = line


_NUM = re.compile(r"^[+-]?(?:\d+\.?\d*(?:[eE][+-]?\d+)?|\.\d+(?:[eE][+-]?\d+)?|inf(?:inity)?|nan)$",
                  re.IGNORECASE)


class _LineReader:
    """tridiag.hpp:115-145: next non-empty line split into doubles."""

    def __init__(self, lines):
        self._lines = lines
        self.line = 0

    def next_row(self, expected: int, what: str) -> list[float]:
        while self.line < len(self._lines):
            text = self._lines[self.line]
            self.line += 1
            if not text.strip(" \t\r\n"):
                continue
            values = []
            for tok in text.split():
                if not _NUM.match(tok):
                    raise ParseError(self.line, f"bad number '{tok}' in {what}")
                values.append(float(tok))
            if len(values) != expected:
                raise ParseError(self.line, f"{what}: expected {expected} values, got {len(values)}")
            return values
        raise ParseError(self.line + 1, f"unexpected end of input reading {what}")


def read_matrix(text: str):
    """tridiag.hpp:171-184"""
    from . import TridiagMatrix
    r = _LineReader(text.splitlines())
    order = r.next_row(1, "matrix order")[0]
    if order < 2 or order != np.floor(order) or order > 1e9:
        raise ParseError(r.line, "matrix order must be an integer >= 2")
    n = int(order)
    sub = r.next_row(n - 1, "sub-diagonal row")
    diag = r.next_row(n, "diagonal row")
    sup = r.next_row(n - 1, "super-diagonal row")
    A = TridiagMatrix(np.array(sub), np.array(diag), np.array(sup))
    A.validate()
    return A


def read_rhs_series(text: str, expect_n: int) -> np.ndarray:
    """tridiag.hpp:198-212"""
    r = _LineReader(text.splitlines())
    header = r.next_row(2, "rhs header")
    if header[0] != float(expect_n):
        raise ParseError(r.line, f"rhs order {int(header[0])} does not match matrix order {expect_n}")
    if header[1] < 1 or header[1] != np.floor(header[1]):
        raise ParseError(r.line, "rhs count must be a positive integer")
    return np.array([r.next_row(expect_n, "rhs row") for _ in range(int(header[1]))])


def _fmt(x: float) -> str:  # "%.17g" (tridiag.hpp:107-111)
    return "%.17g" % x


def write_rhs_series(out, n: int, series: np.ndarray):
    out.write(f"{n} {series.shape[0]}\n")
    for row in series:
        out.write(" ".join(_fmt(v) for v in row) + "\n")


def write_matrix(out, A):
    out.write(f"{A.n()}\n")
    for v in (A.sub, A.diag, A.super):
        out.write(" ".join(_fmt(x) for x in v) + "\n")


def parse_partition(n: int, text: str):
    """Partition::parse (partition.hpp:52-72): comma-separated boundary rows."""
    from . import Partition
    items = []
    for item in text.split(","):
        if not item.strip(" \t"):
            continue
        body = item.lstrip(" \t\n\v\f\r")  # std::stoll skips leading white space only
        if not re.fullmatch(r"[+-]?\d+", body):
            raise ValueError(f"Partition: bad boundary '{item}'")
        v = int(body)
        if v < 0:
            raise ValueError(f"Partition: bad boundary '{item}'")
        items.append(v)
    part = Partition(n, items)
    part.validate()
    return part


def _dense_oracle(A, F: np.ndarray) -> np.ndarray:
    """DenseLU stand-in (main.cpp:92-111): banded LU of A, every RHS."""
    from scipy.linalg import solve_banded
    n = A.n()
    ab = np.zeros((3, n))
    ab[0, 1:] = A.super
    ab[1] = A.diag
    ab[2, :-1] = A.sub
    return solve_banded((1, 1), ab, F.T).T


def cmd_solve(args) -> int:
    from . import SolverError, decompose, Partition, Plan, LAYOUT_S
    try:
        with open(args.matrix) as fh:
            A = read_matrix(fh.read())
    except OSError:
        print(f"parse error: line 0: cannot open matrix file '{args.matrix}'", file=sys.stderr)
        return EXIT_PARSE
    except ParseError as e:
        print(f"parse error: {e}", file=sys.stderr)
        return EXIT_PARSE
    except ValueError as e:  # TridiagMatrix::validate -> std::invalid_argument
        print(f"parse error: {e}", file=sys.stderr)
        return EXIT_PARSE
    try:
        with open(args.rhs) as fh:
            F = read_rhs_series(fh.read(), A.n())
        if args.partition:
            part = parse_partition(A.n(), args.partition)
        else:
            pes = max(args.workers, 1)
            part = Partition(A.n(), []) if pes == 1 else decompose(A.n(), pes).induced_partition()
    except OSError:
        print(f"parse error: line 0: cannot open rhs file '{args.rhs}'", file=sys.stderr)
        return EXIT_PARSE
    except (ParseError, ValueError) as e:
        print(f"parse error: {e}", file=sys.stderr)
        return EXIT_PARSE
    except SolverError as e:  # TooManyPEs from decompose
        print(f"solver error: {e}", file=sys.stderr)
        return EXIT_SOLVER

    try:
        t0 = time.perf_counter()
        plan = Plan(A, part)
        X = plan.solve_host(np.ascontiguousarray(F), layout=LAYOUT_S)
        wall = time.perf_counter() - t0
    except SolverError as e:
        print(f"solver error: {e}", file=sys.stderr)
        return EXIT_SOLVER

    if args.verify:
        want = _dense_oracle(A, F)
        for k in range(F.shape[0]):
            num = float(np.max(np.abs(X[k] - want[k])))
            den = max(float(np.max(np.abs(want[k]))), 1.0)
            if not num <= 1e-9 * den:
                print(f"verification failed on rhs {k}: relative error {num / den}", file=sys.stderr)
                return EXIT_VERIFY

    if args.out:
        with open(args.out, "w") as fh:
            write_rhs_series(fh, A.n(), X)
    else:
        write_rhs_series(sys.stdout, A.n(), X)
    info = plan.info
    # RunStats (run.hpp:42-51): counters of RHS 0 (batch.hpp:69-70), 8 flops
    # per local row (batch.hpp:49)
    stats = json.dumps({"comm_rounds": int(info["comm_rounds"]),
                        "combine_terms": int(info["combine_terms"]),
                        "local_flops": 8 * A.n() if F.shape[0] else 0,
                        "wall_time": wall}, separators=(",", ":"))
    if args.stats:
        with open(args.stats, "w") as fh:
            fh.write(stats + "\n")
    else:
        print(stats, file=sys.stderr)
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="parsweep-b200",
                                 description="batched tridiagonal solves on the GPU")
    ap.add_argument("--workers", type=int, default=1, help="dichotomy blocks when no --partition")
    ap.add_argument("--verify", action="store_true", help="re-check solutions against a dense oracle")
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("solve", help="solve a batch of right-hand sides from files")
    s.add_argument("--matrix", required=True)
    s.add_argument("--rhs", required=True)
    s.add_argument("--partition", default="")
    s.add_argument("--out", default="")
    s.add_argument("--stats", default="")
    args = ap.parse_args(argv)
    return cmd_solve(args)


if __name__ == "__main__":
    sys.exit(main())

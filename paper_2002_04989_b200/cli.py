"""Command-line driver for the B200 path.

Mirrors the reference CLI's hot-path subcommands and output formats
(proj/tools/eigenid.cpp — that binary needs the absent CLI11 header, so this
is a new driver over the same semantics):

    python -m paper_2002_04989_b200.cli full      --random N [--seed S] [--dist gaussian|uniform]
                                                  [--csv F | --mm F] [--out F.csv]
    python -m paper_2002_04989_b200.cli vector    -i I  <source> [--out F.csv] [--signs]
    python -m paper_2002_04989_b200.cli component -i I -j J <source>
    python -m paper_2002_04989_b200.cli bench     --sizes 100 250 ... [--reps R]
                                                  [--task all-vectors] [--seed S]
                                                  [--out records.csv] [--plot-out means.csv]

Engine flags: --batch-size, --workers (accepted, no device meaning),
--log-domain, --degeneracy-tol.  Output: %.12g on stdout, %.17g in CSV files,
row j / column i for `full` (eigenid.cpp:151-176), "j,magnitude" for
`vector` (:139-147), `--signs` prints the signed vector (:129-134,
recover_signs); bench records "n,variant,task,run,seconds,checksum"
(bench.cpp:359-372) and plot data "n,variant,mean_seconds,stddev_seconds"
(bench.cpp:334-357) with variant "gpu-b200".  Exit codes as the reference
(eigenid.cpp:340-350): 0 ok, 1 library error (DegenerateEigenvalue prints the
gap), 2 usage error.
"""
from __future__ import annotations

import argparse
import math
import statistics
import sys
import time

import numpy as np

from . import errors


# ------------------------------------------------------------------ sources
def load_dense_csv(path: str) -> np.ndarray:
    """load_dense_csv (matrix_io.cpp:95-117): one row per line, square."""
    try:
        lines = open(path).read().splitlines()
    except OSError:
        raise errors.Error(f"cannot open {path}")  # FileNotFound
    rows = []
    for ln in lines:
        if not ln:
            continue
        try:
            rows.append([float(t) for t in ln.split(",")])
        except ValueError:
            raise errors.Error(f"cannot parse value in {path}")  # ParseError
    if not rows:
        raise errors.Error(f"no data rows in {path}")
    n = len(rows)
    if any(len(r) != n for r in rows):
        raise errors.DimensionMismatch(f"non-square CSV matrix in {path}")
    return np.array(rows, dtype=np.float64)


def load_matrix_market(path: str) -> np.ndarray:
    """load_matrix_market (matrix_io.cpp:119-167): coordinate real symmetric,
    lower triangle, 1-based."""
    try:
        lines = open(path).read().splitlines()
    except OSError:
        raise errors.Error(f"cannot open {path}")
    if not lines or lines[0].split()[:5] != ["%%MatrixMarket", "matrix", "coordinate",
                                            "real", "symmetric"]:
        raise errors.Error(f"unsupported MatrixMarket header in {path}")
    body = [ln for ln in lines[1:] if ln and not ln.startswith("%")]
    n, cols, nnz = (int(t) for t in body[0].split())
    if n != cols:
        raise errors.DimensionMismatch(f"MatrixMarket matrix is not square in {path}")
    a = np.zeros((n, n))
    for ln in body[1:]:
        r, c, v = ln.split()
        r, c = int(r) - 1, int(c) - 1
        if c > r:
            raise errors.Error(f"upper-triangle entry in symmetric file {path}")
        a[r, c] = a[c, r] = float(v)
    if len(body) - 1 != nnz:
        raise errors.Error(f"entry count mismatch in {path}")
    return a


def load_source(args) -> np.ndarray:
    from .engine import SymmetricMatrix
    if args.csv:
        return SymmetricMatrix.build(*_flat(load_dense_csv(args.csv))).array()
    if args.mm:
        return SymmetricMatrix.build(*_flat(load_matrix_market(args.mm))).array()
    if args.random and args.random > 0:
        return random_symmetric(args.seed, args.random, args.dist)
    raise errors.ConfigError("no matrix source given: use --csv, --mm or --random")


def _flat(a):
    return a.shape[0], a.reshape(-1)


def random_symmetric(seed: int, n: int, dist: str = "gaussian") -> np.ndarray:
    from .engine import random_symmetric as gen
    return gen(seed, n, dist)


def splitmix64(x: int) -> int:
    """bench.cpp:78-83."""
    m = (1 << 64) - 1
    x = (x + 0x9E3779B97F4A7C15) & m
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & m
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & m
    return x ^ (x >> 31)


def _engine(args):
    from .engine import IdentityConfig, IdentityEngine
    if args.batch_size < 1:
        raise errors.ConfigError("batch size must be >= 1")
    return IdentityEngine(IdentityConfig(
        batch_size=args.batch_size, workers=args.workers,
        degeneracy_tol=args.degeneracy_tol,
        evaluation="log-domain" if args.log_domain else "paired-batched"))


def fmt12(v: float) -> str:
    return f"{v:.12g}"


# ------------------------------------------------------------------ commands
def run_full(args) -> int:
    a = load_source(args)
    n = a.shape[0]
    m = _engine(args).all_magnitudes(a).reshape(n, n)
    if args.out:
        with open(args.out, "w") as f:
            for j in range(n):
                f.write(",".join(f"{v:.17g}" for v in m[j]) + "\n")
    else:
        for j in range(n):
            print(",".join(fmt12(v) for v in m[j]))
    return 0


def run_vector(args) -> int:
    a = load_source(args)
    n = a.shape[0]
    if args.i >= n:
        return usage_error(f"index i={args.i} out of range for n = {n}")
    v = _engine(args).vector_magnitudes(a, args.i)
    if args.signs:  # eigenid.cpp:129-134: signed vector, %.12g per line
        from .engine import eigenvalues, recover_signs
        s = eigenvalues(a)
        for x in recover_signs(a, args.i, v, s[args.i]):
            print(fmt12(x))
        return 0
    if args.out:
        with open(args.out, "w") as f:
            f.write("j,magnitude\n")
            for j in range(n):
                f.write(f"{j},{v[j]:.17g}\n")
    else:
        for x in v:
            print(fmt12(x))
    return 0


def run_component(args) -> int:
    a = load_source(args)
    n = a.shape[0]
    if args.i >= n or args.j >= n:
        return usage_error(f"indices (i={args.i}, j={args.j}) out of range for n = {n}")
    eng = _engine(args)
    f = eng.log_domain_magnitude if args.log_domain else eng.component_magnitude
    print(fmt12(f(a, args.i, args.j)[0]))
    return 0


TASKS = ("single-component", "single-vector", "all-vectors")


def run_bench(args) -> int:
    """run_benchmark (bench.cpp:190-285) for the GPU variant: one seeded
    matrix per size (seed ^ splitmix64(n)), an untimed warm-up with the
    solve-count check (n+1 for vector/all tasks, 2 for single-component),
    then timed repetitions with the task checksum."""
    if not args.sizes:
        raise errors.ConfigError("size list is empty")
    if any(n < 2 for n in args.sizes):
        raise errors.ConfigError("benchmark sizes must be >= 2")
    if args.reps < 1:
        raise errors.ConfigError("repetitions must be >= 1")
    if args.task not in TASKS:
        raise errors.ConfigError(f"unknown task '{args.task}'")
    eng = _engine(args)
    records = []
    for n in args.sizes:
        a = random_symmetric(args.seed ^ splitmix64(n), n, args.dist)
        i, j = n // 2, n // 3

        def task():
            if args.task == "single-component":
                return eng.component_magnitude(a, i, j)[0]
            if args.task == "single-vector":
                return float(np.sum(eng.vector_magnitudes(a, i)))
            return float(np.sum(eng.all_magnitudes(a)))

        eng.reset_solve_count()
        task()
        want = 2 if args.task == "single-component" else n + 1
        if eng.eigenvalue_solve_count() != want:
            raise errors.InternalInconsistency(
                f"eigenvalue solve count at n = {n} is "
                f"{eng.eigenvalue_solve_count()}, expected {want}")
        for run in range(args.reps):
            t0 = time.perf_counter()
            checksum = task()
            records.append((n, "gpu-b200", args.task, run,
                            time.perf_counter() - t0, checksum))
        if not math.isfinite(checksum):
            raise errors.Error(f"non-finite checksum at n = {n}")
    if args.out:
        with open(args.out, "w") as f:
            f.write("n,variant,task,run,seconds,checksum\n")
            for r in records:
                f.write(f"{r[0]},{r[1]},{r[2]},{r[3]},{r[4]:.6f},{r[5]:.17g}\n")
    if args.plot_out:
        with open(args.plot_out, "w") as f:
            f.write("n,variant,mean_seconds,stddev_seconds\n")
            for n in args.sizes:
                ts = [r[4] for r in records if r[0] == n]
                mean = sum(ts) / len(ts)
                var = sum(t * t for t in ts) / len(ts) - mean * mean
                f.write(f"{n},gpu-b200,{mean:.17g},{math.sqrt(max(var, 0.0)):.17g}\n")
    for n in args.sizes:
        ts = [r[4] for r in records if r[0] == n]
        print(f"n={n} gpu-b200 mean {statistics.mean(ts):.6f} s")
    return 0


def usage_error(msg: str) -> int:
    print(f"usage error: {msg}", file=sys.stderr)
    return 2


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(
        prog="eigenid-b200",
        description="eigenvector component magnitudes via eigenvalues of matrix minors (B200)")
    sub = ap.add_subparsers(dest="cmd", required=True)

    def source(p):
        g = p.add_mutually_exclusive_group()
        g.add_argument("--csv", help="dense CSV matrix file")
        g.add_argument("--mm", help="MatrixMarket symmetric matrix file")
        g.add_argument("--random", type=int, help="random symmetric matrix of size N")
        p.add_argument("--seed", type=int, default=0)
        p.add_argument("--dist", choices=["gaussian", "uniform"], default="gaussian")

    def engine(p):
        p.add_argument("--batch-size", type=int, default=64)
        p.add_argument("--workers", type=int, default=0)
        p.add_argument("--log-domain", action="store_true")
        p.add_argument("--degeneracy-tol", type=float, default=1e-12)

    p = sub.add_parser("component")
    source(p), engine(p)
    p.add_argument("-i", type=int, required=True)
    p.add_argument("-j", type=int, required=True)
    p = sub.add_parser("vector")
    source(p), engine(p)
    p.add_argument("-i", type=int, required=True)
    p.add_argument("--out")
    p.add_argument("--signs", action="store_true",
                   help="recover component signs from the row equations")
    p = sub.add_parser("full")
    source(p), engine(p)
    p.add_argument("--out")
    p = sub.add_parser("bench")
    engine(p)
    p.add_argument("--sizes", type=int, nargs="+", default=[2, 100, 250, 500, 1000])
    p.add_argument("--reps", type=int, default=10)
    p.add_argument("--task", default="all-vectors")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--dist", choices=["gaussian", "uniform"], default="gaussian")
    p.add_argument("--out")
    p.add_argument("--plot-out")
    return ap


def main(argv=None) -> int:
    ap = build_parser()
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 2
    try:
        return {"full": run_full, "vector": run_vector, "component": run_component,
                "bench": run_bench}[args.cmd](args)
    except errors.ConfigError as e:
        return usage_error(str(e))
    except errors.DegenerateEigenvalue as e:
        print(f"error: degenerate eigenvalue (gap {e.gap():g}): {e}", file=sys.stderr)
        return 1
    except errors.Error as e:
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())

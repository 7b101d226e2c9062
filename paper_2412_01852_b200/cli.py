"""``rotbench``-compatible command line for the B200 path.

Mirrors the reference's ``rotbench run`` / ``rotbench verify`` (cli.py:166-260) for the
GPU algorithms registered in :mod:`verification` (``cuda``, ``cuda-naive``):

* ``run``  times an algorithm on ``make_inputs(m, n, k, seed)`` (best of ``--reps``) and
  writes the reference's CSV (``n,Flops`` in GFLOP/s; ``--csv-extended`` adds the
  reference's extra columns plus the device-side kernel time and its fraction of the
  live FMA-pipe peak). ``--timing host`` (default, the reference's semantics) times the
  whole call on host data; ``--timing device`` times the packed kernel on resident data.
  Small cases are verified against the independent ``cuda-naive`` kernel (the reference
  verifies against its own ``apply_naive``); a failed check exits 1.
* ``verify``  the reference's equivalence grids (cli.py:243-278): criterion 1, the
  bitwise grid (verification.py:161-195) in strict arithmetic, ``cuda`` against the
  independent ``cuda-naive`` kernel; criterion 2, the explicit-Q chain
  (verification.py:198-219), both algorithms against ``A0 @ Q`` with Q accumulated on
  the host. ``--perturb-kernel`` sets ``ROTSEQ_PERTURB_KERNEL`` for the run (cli.py:244-245)
  so the kernel path's output is off by one ulp and verify must exit 1.

Usage: ``python -m paper_2412_01852_b200.cli run --algo cuda --n 4096 --k 192``.
Argument errors and ``ValueError`` exit with status 2, as in the reference (cli.py:372-374).
"""

from __future__ import annotations

import argparse
import math
import os
import sys
import time

from .compare import compare
from .core import Order, Side, TransformKind, flops_applied, make_inputs
from .verification import ALGORITHMS, FAULT_ENV, bitwise_grid, oracle_grid, run_variant

VERIFY_SIZE_LIMIT = 512 * 512  # the reference verifies runs up to this many elements


def _cpu_knobs(p: argparse.ArgumentParser) -> None:
    """The reference's CPU cache/thread flags (cli.py:93-117): accepted so command lines
    port unchanged, and ignored (the GPU tiling is chosen by the library)."""
    for flag in ("--mr", "--kr", "--nb", "--kb", "--mb", "--T1", "--T2", "--T3", "--S", "--threads"):
        p.add_argument(flag, type=int, help=argparse.SUPPRESS)
    p.add_argument("--config", help=argparse.SUPPRESS)


def _parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="rotbench-b200", description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="command", required=True)
    run = sub.add_parser("run", help="time one algorithm, CSV out")
    run.add_argument("--algo", choices=ALGORITHMS, default="cuda")
    run.add_argument("--n", type=int)
    run.add_argument("--m", type=int)
    run.add_argument("--k", type=int, default=180)
    run.add_argument("--sweep", type=int, nargs="+", help="square sizes m = n")
    run.add_argument("--seed", type=int, default=0)
    run.add_argument("--reps", type=int, default=3)
    run.add_argument("--kind", choices=("rotation", "reflector"), default="rotation")
    run.add_argument("--strict-arith", choices=("on", "off"), default="off")
    run.add_argument("--side", choices=("right", "left"), default="right")
    run.add_argument("--order", choices=("forward", "reverse"), default="forward")
    run.add_argument("--timing", choices=("host", "device"), default="host")
    run.add_argument("--csv", help="write the CSV here instead of stdout")
    run.add_argument("--csv-extended", action="store_true")
    run.add_argument("--verify-all", action="store_true", help="verify every size, not only small ones")
    _cpu_knobs(run)
    ver = sub.add_parser("verify", help="equivalence grids (bitwise + explicit Q), exit 1 on failure")
    ver.add_argument("--quick", action="store_true")
    ver.add_argument("--seed", type=int, default=0)
    ver.add_argument("--kind", choices=("rotation", "reflector"))
    ver.add_argument("--perturb-kernel", action="store_true", help=argparse.SUPPRESS)
    _cpu_knobs(ver)
    return ap


def _device_time(A0, seq, kind, fast, side, order, reps):
    """Best packed-kernel time (s) on resident device data."""
    import torch

    from .apply import PackedSequence

    dev = torch.device("cuda", torch.cuda.current_device())
    dA = torch.from_numpy(A0).to(dev)  # keeps the column-major strides
    C = torch.from_numpy(seq.C).to(dev)
    S = torch.from_numpy(seq.S).to(dev)
    packed = PackedSequence((C, S), dA.shape, kind=kind, side=side, order=order, device=dev, fast_only=fast)
    packed.apply(dA, fast=fast)
    best = math.inf
    for _ in range(max(reps, 1)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        packed.apply(dA, fast=fast)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    return best


def cmd_run(args) -> int:
    from . import _lib

    if args.sweep is not None:
        sizes = [(s, s, args.k) for s in args.sweep]
    else:
        if args.n is None:
            raise ValueError("run needs --n (or --sweep)")
        sizes = [(args.m if args.m is not None else args.n, args.n, args.k)]
    kind = TransformKind.REFLECTOR if args.kind == "reflector" else TransformKind.ROTATION
    side = Side(args.side)
    order = Order(args.order)
    fast = args.strict_arith == "off"
    peak = None
    records = []
    any_fail = False
    for m, n, k in sizes:
        A0, seq = make_inputs(m, n, k, args.seed)
        if side is Side.LEFT:
            from .core import generate_sequence

            seq = generate_sequence(m, k, args.seed + 1)

        def one_rep():
            work = A0.copy(order="F")
            t0 = time.perf_counter()
            run_variant(args.algo, work, seq, kind, fast=fast, side=side, order=order)
            return time.perf_counter() - t0, work

        one_rep()  # warm-up (library load, first-touch of the stream-ordered pool)
        best, last = math.inf, None
        for _ in range(max(args.reps, 1)):
            dt, last = one_rep()
            best = min(best, dt)
        kernel_s = None
        if args.timing == "device" or args.csv_extended:
            kernel_s = _device_time(A0, seq, kind, fast, side, order, args.reps)
        secs = kernel_s if args.timing == "device" else best
        verified = None
        if args.verify_all or m * n <= VERIFY_SIZE_LIMIT:
            ref = A0.copy(order="F")
            run_variant("cuda-naive" if args.algo == "cuda" else "cuda", ref, seq, kind, fast=fast, side=side,
                        order=order)
            verified = bool(compare(ref, last, tol_profile="fast" if fast else "strict", k=k).passed)
            any_fail = any_fail or not verified
        fl = flops_applied(m, n, k, side)
        rec = dict(algo=args.algo, m=m, n=n, k=k, reps=args.reps, seconds=secs, gflops=fl / secs / 1e9,
                   verified=verified)
        if kernel_s is not None:
            if peak is None:
                peak = _lib.fma_peak_tflops(_lib.DTYPE_F64)
            rec["kernel_seconds"] = kernel_s
            rec["peak_frac"] = fl / kernel_s / 1e12 / peak
        records.append(rec)
        print(f"{args.algo:10s} m={m} n={n} k={k}: {secs * 1e3:.3f} ms  {rec['gflops']:.1f} GF/s"
              + (f"  verified={verified}" if verified is not None else ""), file=sys.stderr)
    sink = open(args.csv, "w") if args.csv else sys.stdout
    try:
        if args.csv_extended:
            sink.write("n,Flops,algo,m,k,threads,reps,seconds,verified,kernel_seconds,peak_frac\n")
            for r in records:
                sink.write(f"{r['n']},{r['gflops']:.9g},{r['algo']},{r['m']},{r['k']},1,{r['reps']},"
                           f"{r['seconds']:.9g},{r['verified']},{r['kernel_seconds']:.9g},{r['peak_frac']:.6f}\n")
        else:
            sink.write("n,Flops\n")
            for r in records:
                sink.write(f"{r['n']},{r['gflops']:.9g}\n")
    finally:
        if sink is not sys.stdout:
            sink.close()
    return 1 if any_fail else 0


def cmd_verify(args) -> int:
    """Criteria 1 and 2 of the reference's verify (cli.py:243-278)."""
    if args.perturb_kernel:
        os.environ[FAULT_ENV] = "1"
    try:
        kinds = ((TransformKind.ROTATION, TransformKind.REFLECTOR) if args.kind is None
                 else ((TransformKind.REFLECTOR,) if args.kind == "reflector" else (TransformKind.ROTATION,)))
        total, failures = 0, []
        for kind in kinds:
            for case in bitwise_grid(kind, quick=args.quick, seed=args.seed):
                total += 1
                if not case.ok:
                    failures.append(case)
                    print(case, file=sys.stderr)
            for case in oracle_grid(kind, seed=args.seed):
                total += 1
                if not case.ok:
                    failures.append(case)
                    print(case, file=sys.stderr)
        print(f"verify: {total - len(failures)}/{total} cases passed")
        if failures:
            worst = failures[0]
            print(f"verify: FIRST FAILURE {worst.algo} [{worst.config}] kind={worst.kind} "
                  f"m={worst.m} n={worst.n} k={worst.k}", file=sys.stderr)
            return 1
        return 0
    finally:
        if args.perturb_kernel:
            os.environ.pop(FAULT_ENV, None)


def main(argv=None) -> int:
    args = _parser().parse_args(argv)
    try:
        return cmd_run(args) if args.command == "run" else cmd_verify(args)
    except (ValueError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())

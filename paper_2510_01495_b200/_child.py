"""Fresh-process worker for overhead.estimate_overhead (reference _child.py:13-44).

Builds the operands on the host, then times the first call and ``--trials`` calls after it with
the native clock and writes (trial, is_warmup, elapsed_s) rows to the CSV given as the first
argument. Exit 0 on success; any failure exits nonzero so the parent discards the repeat.
"""

import argparse
import csv
import sys


def _operands(experiment, size, seed, density, mode):
    from . import synth
    ts = synth.derive_trial_seed(seed, 0, 0)
    if experiment == "dot":
        return (synth.gen_vector(synth.GenSpec(synth.derive_arg_seed(ts, 0), "vector", (size,))),
                synth.gen_vector(synth.GenSpec(synth.derive_arg_seed(ts, 1), "vector", (size,))))
    if experiment == "matvec":
        return (synth.gen_matrix(synth.GenSpec(synth.derive_arg_seed(ts, 0), "matrix", (size, size))),
                synth.gen_vector(synth.GenSpec(synth.derive_arg_seed(ts, 1), "vector", (size,))))
    k = (mode if mode is not None else 3) - 1
    t = synth.gen_sparse3(synth.GenSpec(synth.derive_arg_seed(ts, 0), "sparse3", (size,) * 3,
                                        density if density is not None else 0.001))
    x = synth.gen_vector(synth.GenSpec(synth.derive_arg_seed(ts, 1), "vector", (size,)))
    return t.subs, t.vals, t.shape, x, k


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="tk-overhead-child")
    ap.add_argument("out")
    ap.add_argument("--experiment", required=True, choices=["dot", "matvec", "ttv"])
    ap.add_argument("--size", type=int, required=True)
    ap.add_argument("--trials", type=int, required=True)
    ap.add_argument("--seed", type=int, required=True)
    ap.add_argument("--density", type=float, default=None)
    ap.add_argument("--mode", type=int, default=None)
    a = ap.parse_args(argv)
    ops = _operands(a.experiment, a.size, a.seed, a.density, a.mode)
    # deferred: the timed first call sees a process that has only imported the package
    from . import _kernels as K
    call = {"dot": lambda: K.dot_timed(*ops)[1], "matvec": lambda: K.matvec_timed(*ops)[1],
            "ttv": lambda: K.ttv_timed(*ops)[1]}[a.experiment]
    rows = [(0, 1, call())]
    rows += [(i + 1, 0, call()) for i in range(a.trials)]
    with open(a.out, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["trial", "is_warmup", "elapsed_s"])
        for r in rows:
            w.writerow([r[0], r[1], f"{r[2]:.17g}"])
    return 0


if __name__ == "__main__":
    try:
        code = main()
    except Exception as exc:  # the parent discards this repeat
        print(f"tk-overhead-child: {exc}", file=sys.stderr)
        code = 1
    sys.exit(code)

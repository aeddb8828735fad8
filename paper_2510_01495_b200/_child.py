"""Interpreter shim for the reference's fresh-process harness children.

The reference's first-call overhead estimator (/root/reference/pkg/hostbench/src/tenhost/
overhead.py:76-175) launches ``[sys.executable, "-m", "tenhost._child", out, --impl LABEL, ...]``
and the child resolves LABEL in the reference's registry (tenhost/_child.py:13-44).  Labels live
in process memory, so a child only knows ``b200`` if something registers it first.  This shim is
that something: ``python -m paper_2510_01495_b200._child -m tenhost._child ...`` registers the
B200 labels (``registry.register``) and then runs the requested module exactly as ``-m`` would.
Registration imports the packages and loads libtk_b200.so but creates no CUDA context, so the
child's first timed call still pays the full first-call cost being estimated.
"""

import runpy
import sys


def main(argv) -> None:
    if len(argv) < 2 or argv[0] != "-m":
        raise SystemExit("usage: python -m paper_2510_01495_b200._child -m MODULE [ARGS...]")
    module = argv[1]
    from .registry import register
    register()
    sys.argv = [module] + list(argv[2:])
    runpy.run_module(module, run_name="__main__", alter_sys=True)


if __name__ == "__main__":
    main(sys.argv[1:])

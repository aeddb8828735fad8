"""Exception module for the shim ``tenkern`` package in oracle/_ref/.

The reference's compiled kernel module imports DimensionError, ModeError and
OrderError from ``tenkern.errors`` at import time (pkg/src/tenkern/_ckernels.pyx:24).
The GPU box has no /root/reference, so oracle/Makefile installs this file as
``oracle/_ref/tenkern/errors.py`` next to the compiled extension.  The class
names and bases follow pkg/src/tenkern/errors.py:4-37.
"""


class TenkernError(Exception):
    pass


class DimensionError(TenkernError, ValueError):
    pass


class ModeError(TenkernError, ValueError):
    pass


class OrderError(TenkernError, ValueError):
    pass

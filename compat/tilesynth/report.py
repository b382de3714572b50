"""Compat alias: reference module ``tilesynth.report`` -> ``paper_2504_16214_b200.tilesynth.reporting``."""
import sys as _sys

from paper_2504_16214_b200.tilesynth import reporting as _m

_sys.modules[__name__] = _m

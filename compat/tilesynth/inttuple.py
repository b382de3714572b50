"""Compat alias: reference module ``tilesynth.inttuple`` -> ``paper_2504_16214_b200.tilesynth.ituple``."""
import sys as _sys

from paper_2504_16214_b200.tilesynth import ituple as _m

_sys.modules[__name__] = _m

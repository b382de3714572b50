"""Compat alias: reference module ``tilesynth.inttuple`` -> ``paper_2504_16214_b200.tilesynth.tuples``."""
import sys as _sys

from paper_2504_16214_b200.tilesynth import tuples as _m

_sys.modules[__name__] = _m

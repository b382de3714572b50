"""Compat alias: reference module ``tilesynth.tv`` -> ``paper_2504_16214_b200.tilesynth.algebra``."""
import sys as _sys

from paper_2504_16214_b200.tilesynth import algebra as _m

_sys.modules[__name__] = _m

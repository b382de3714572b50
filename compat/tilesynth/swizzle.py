"""Compat alias: reference module ``tilesynth.swizzle`` -> ``paper_2504_16214_b200.tilesynth.banking``."""
import sys as _sys

from paper_2504_16214_b200.tilesynth import banking as _m

_sys.modules[__name__] = _m

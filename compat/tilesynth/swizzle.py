"""Compat alias: reference module ``tilesynth.swizzle`` -> ``paper_2504_16214_b200.tilesynth.banks``."""
import sys as _sys

from paper_2504_16214_b200.tilesynth import banks as _m

_sys.modules[__name__] = _m

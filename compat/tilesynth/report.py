"""Compat alias: reference module ``tilesynth.report`` -> ``paper_2504_16214_b200.tilesynth.frontend``."""
import sys as _sys

from paper_2504_16214_b200.tilesynth import frontend as _m

_sys.modules[__name__] = _m

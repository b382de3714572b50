"""Compat alias: reference module ``tilesynth.errors`` -> ``paper_2504_16214_b200.tilesynth.errors``."""
import sys as _sys

from paper_2504_16214_b200.tilesynth import errors as _m

_sys.modules[__name__] = _m

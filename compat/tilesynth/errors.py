"""Compat alias: reference module ``tilesynth.errors`` -> ``paper_2504_16214_b200.tilesynth.exceptions``."""
import sys as _sys

from paper_2504_16214_b200.tilesynth import exceptions as _m

_sys.modules[__name__] = _m

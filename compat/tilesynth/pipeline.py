"""Compat alias: reference module ``tilesynth.pipeline`` -> ``paper_2504_16214_b200.tilesynth.driver``."""
import sys as _sys

from paper_2504_16214_b200.tilesynth import driver as _m

_sys.modules[__name__] = _m

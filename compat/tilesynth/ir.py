"""Compat alias: reference module ``tilesynth.ir`` -> ``paper_2504_16214_b200.tilesynth.tileprog``."""
import sys as _sys

from paper_2504_16214_b200.tilesynth import tileprog as _m

_sys.modules[__name__] = _m

"""Compat alias: reference module ``tilesynth.tv`` -> ``paper_2504_16214_b200.tilesynth.tvmap``."""
import sys as _sys

from paper_2504_16214_b200.tilesynth import tvmap as _m

_sys.modules[__name__] = _m

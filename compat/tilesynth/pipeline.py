"""Compat alias: reference module ``tilesynth.pipeline`` -> ``paper_2504_16214_b200.tilesynth.synthesize``."""
import sys as _sys

from paper_2504_16214_b200.tilesynth import synthesize as _m

_sys.modules[__name__] = _m

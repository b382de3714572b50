"""Compat alias: reference module ``tilesynth.synth`` -> ``paper_2504_16214_b200.tilesynth.propagation``."""
import sys as _sys

from paper_2504_16214_b200.tilesynth import propagation as _m

_sys.modules[__name__] = _m

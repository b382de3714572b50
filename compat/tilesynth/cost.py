"""Compat alias: reference module ``tilesynth.cost`` -> ``paper_2504_16214_b200.tilesynth.explore``."""
import sys as _sys

from paper_2504_16214_b200.tilesynth import explore as _m

_sys.modules[__name__] = _m

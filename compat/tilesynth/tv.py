"""Compat alias: reference module ``tilesynth.tv`` -> ``paper_2504_16214_b200.tilesynth.tvl``."""
import sys as _sys

from paper_2504_16214_b200.tilesynth import tvl as _m

_sys.modules[__name__] = _m

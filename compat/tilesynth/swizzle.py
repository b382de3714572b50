"""Compat alias: reference module ``tilesynth.swizzle`` -> ``paper_2504_16214_b200.tilesynth.bankmodel``."""
import sys as _sys

from paper_2504_16214_b200.tilesynth import bankmodel as _m

_sys.modules[__name__] = _m

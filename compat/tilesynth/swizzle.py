"""Compat alias: reference module ``tilesynth.swizzle`` -> ``paper_2504_16214_b200.tilesynth.smem_plan``."""
import sys as _sys

from paper_2504_16214_b200.tilesynth import smem_plan as _m

_sys.modules[__name__] = _m

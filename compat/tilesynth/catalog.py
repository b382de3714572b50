"""Compat alias: reference module ``tilesynth.catalog`` -> ``paper_2504_16214_b200.tilesynth.isa_table``."""
import sys as _sys

from paper_2504_16214_b200.tilesynth import isa_table as _m

_sys.modules[__name__] = _m

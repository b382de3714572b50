"""Compat alias: reference module ``tilesynth.catalog`` -> ``paper_2504_16214_b200.tilesynth.instr_catalog``."""
import sys as _sys

from paper_2504_16214_b200.tilesynth import instr_catalog as _m

_sys.modules[__name__] = _m

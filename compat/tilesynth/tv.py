"""Compat alias: reference module ``tilesynth.tv`` -> ``paper_2504_16214_b200.tilesynth.thread_value``."""
import sys as _sys

from paper_2504_16214_b200.tilesynth import thread_value as _m

_sys.modules[__name__] = _m

"""Compat alias: reference module ``tilesynth.cost`` -> ``paper_2504_16214_b200.tilesynth.latency_model``."""
import sys as _sys

from paper_2504_16214_b200.tilesynth import latency_model as _m

_sys.modules[__name__] = _m

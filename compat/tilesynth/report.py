"""Compat alias: reference module ``tilesynth.report`` -> ``paper_2504_16214_b200.tilesynth.report_json``."""
import sys as _sys

from paper_2504_16214_b200.tilesynth import report_json as _m

_sys.modules[__name__] = _m

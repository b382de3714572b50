"""Compat package: exposes the re-implemented synthesizer under the reference's module names
(``tilesynth.layout``, ``tilesynth.synth`` ...) so the reference's own test-suite can run against it
unmodified (tests/test_tilesynth_parity.py::test_reference_suite_against_reimplementation)."""
import os as _os
import sys as _sys

_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.dirname(_os.path.abspath(__file__)))))

from paper_2504_16214_b200.tilesynth import *  # noqa: E402,F401,F403
from paper_2504_16214_b200.tilesynth import __all__, __version__  # noqa: E402,F401

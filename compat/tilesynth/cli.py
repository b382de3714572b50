"""Compat alias: reference module ``tilesynth.cli`` -> ``paper_2504_16214_b200.tilesynth.frontend``
(also runnable as ``python -m tilesynth.cli``)."""
import sys as _sys

from paper_2504_16214_b200.tilesynth import frontend as _m

if __name__ == "__main__":
    _sys.exit(_m.main())
else:
    _sys.modules[__name__] = _m

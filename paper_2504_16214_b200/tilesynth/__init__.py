"""Layout synthesis for tile programs (host side of the W4A16 path) -- a re-implementation of the
reference ``tilesynth`` API (``/root/reference/pkg/src/tilesynth/__init__.py:16-58``) whose chosen
thread-value, shared-memory and swizzle layouts, instruction choices, costs and JSON reports are
bit-identical to the reference on the same programs (tests/test_tilesynth_parity.py).

Module map (reference -> here): inttuple -> tuples, errors -> exceptions, layout -> algebra,
tv -> thread_value, swizzle -> banks, ir -> program, catalog -> isa, synth -> propagation,
smem -> smem_synth, cost -> latency, pipeline -> driver, report -> reporting, cli -> cli.
``compat/tilesynth`` re-exports them under the reference module names.
"""
from .algebra import (Layout, coalesce, complement, compose, concat, dim_restrict, inverse, parse_layout,
                      restrict_first_mode)
from .banks import Swizzle, bank_conflicts
from .driver import SynthesisResult, synthesize_program
from .isa import Catalog, Instruction, builtin_catalog_path, load_catalog
from .program import ProgramGraph, parse_program, validate
from .propagation import SynthesisConfig
from .thread_value import TvLayout

__version__ = "0.1.0"

__all__ = [
    "Catalog", "Instruction", "Layout", "ProgramGraph", "SynthesisConfig", "SynthesisResult", "Swizzle", "TvLayout",
    "bank_conflicts", "builtin_catalog_path", "coalesce", "complement", "compose", "concat", "dim_restrict",
    "inverse", "load_catalog", "parse_layout", "parse_program", "restrict_first_mode", "synthesize_program",
    "validate",
]

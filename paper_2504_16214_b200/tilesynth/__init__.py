"""Layout synthesis for tile programs -- the host side of the W4A16 path, written for this repository.

It answers the reference's API (``/root/reference/pkg/src/tilesynth/__init__.py:16-58``) with the same
results: chosen thread-value, shared-memory and swizzle layouts, instructions, costs and JSON reports
are byte-identical to the reference's on the same programs (tests/test_tilesynth_parity.py). Modules:

* ``nested``          nested integer tuples (colex digits, text form)
* ``layout_algebra``  ``Layout`` and its algebra; numpy tables of whole maps
* ``tvl``             thread-value layouts with cached position grids
* ``banking``         swizzles and the vectorised 32-bank conflict model
* ``tile_ir``         program text format, validation, liveness, components
* ``instr_catalog``   instruction models (``data/*.cat``) and queries
* ``tv_solver``       anchors and round-based constraint propagation
* ``smem_layout``     shared-memory constraints, unification, materialisation, swizzle choice
* ``search``          the candidate walk with per-component memoisation
* ``latency_model``   the issue / completion latency model and ranking
* ``synthesize``      ``synthesize_program``;  ``report_json`` reports;  ``cli`` the command line

``compat/tilesynth`` maps the reference's module names onto these.
"""
from .banking import Swizzle, bank_conflicts
from .instr_catalog import Catalog, Instruction, builtin_catalog_path, load_catalog
from .layout_algebra import (Layout, coalesce, complement, compose, concat, dim_restrict, inverse, parse_layout,
                             restrict_first_mode)
from .synthesize import SynthesisResult, synthesize_program
from .tile_ir import ProgramGraph, parse_program, validate
from .tv_solver import SynthesisConfig
from .tvl import TvLayout

__version__ = "0.1.0"

__all__ = [
    "Catalog", "Instruction", "Layout", "ProgramGraph", "SynthesisConfig", "SynthesisResult", "Swizzle", "TvLayout",
    "bank_conflicts", "builtin_catalog_path", "coalesce", "complement", "compose", "concat", "dim_restrict",
    "inverse", "load_catalog", "parse_layout", "parse_program", "restrict_first_mode", "synthesize_program",
    "validate",
]

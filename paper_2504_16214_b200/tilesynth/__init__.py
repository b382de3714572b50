"""Layout synthesis for tile programs -- the host side of the W4A16 path, written for this repository.

It answers the reference's API (``/root/reference/pkg/src/tilesynth/__init__.py:16-58``) with the same
results: chosen thread-value, shared-memory and swizzle layouts, instructions, costs and JSON reports
are byte-identical to the reference's on the same programs (tests/test_tilesynth_parity.py). Modules:

* ``ituple``      nested integer tuples (iterative walks, token-machine parser)
* ``algebra``     ``Layout`` over flat run lists, interval-based composition, numpy tables; thread-value
                  layouts with whole-domain position grids
* ``tileprog``    program text format (handler table), validation rules, liveness, components
* ``isa_table``   instruction catalogs (``data/*.cat``) and queries
* ``layout_flow`` anchors and round-based constraint propagation
* ``smem_plan``   swizzles and the array-at-a-time 32-bank conflict model; shared-memory constraints,
                  unification, materialisation, swizzle choice
* ``explore``     the candidate walk (per-component memoisation), ``synthesize_program``, the issue /
                  completion latency model (tensor scoreboard) and ranking
* ``frontend``    JSON / text reports, ``--explain`` and the ``tilesynth`` command line

``compat/tilesynth`` maps the reference's module names onto these.
"""
from . import algebra as _algebra, explore as _explore, isa_table as _isa, layout_flow as _flow, smem_plan as _smem
from . import tileprog as _prog

__version__ = "0.1.0"

# public name -> the module that defines it (the reference's export list, tilesynth/__init__.py:16-58)
_EXPORTS = {
    _algebra: "Layout TvLayout coalesce complement compose concat dim_restrict inverse parse_layout restrict_first_mode",
    _smem: "Swizzle bank_conflicts",
    _explore: "SynthesisResult synthesize_program",
    _isa: "Catalog Instruction builtin_catalog_path load_catalog",
    _flow: "SynthesisConfig",
    _prog: "ProgramGraph parse_program validate",
}
globals().update({name: getattr(mod, name) for mod, names in _EXPORTS.items() for name in names.split()})
__all__ = sorted(name for names in _EXPORTS.values() for name in names.split())

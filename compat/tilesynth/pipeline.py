"""Compat module: reference module ``tilesynth.pipeline`` = this repository's ``explore``
(``synthesize_program`` / ``SynthesisResult`` live next to the search)."""
from paper_2504_16214_b200.tilesynth.explore import SynthesisResult, synthesize_program  # noqa: F401

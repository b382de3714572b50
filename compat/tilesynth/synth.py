"""Compat module: reference module ``tilesynth.synth`` = this repository's ``layout_flow`` (anchors,
propagation) + ``explore`` (candidates, shared / staging buffers, the search walk)."""
from paper_2504_16214_b200.tilesynth.explore import (PRUNE as _PRUNE_ERRORS, Candidate, _copy_choice_points,  # noqa: F401
                                                     _staging_instructions, _synthesize_shared, _synthesize_staging,
                                                     evaluate_assignment, expand_search)
from paper_2504_16214_b200.tilesynth.layout_flow import (PropagationState, RearrangePatch, SlotKey,  # noqa: F401
                                                         SynthesisConfig, TvConstraint, _anchor_copy, _warp_grid,
                                                         build_constraints, coalesced_access_layout,
                                                         init_gemm_anchor, propagate, reduce_projection, slot_for,
                                                         solve_copy, solve_reduce)
from paper_2504_16214_b200.tilesynth.algebra import TvLayout, restrict_tv, tv_from_mode_lists  # noqa: F401

"""B200-native re-build of Hexcute's (arXiv 2504.16214) W4A16 MoE hot path.

* :mod:`paper_2504_16214_b200.tilesynth` -- the layout-synthesis host API (same names and results as
  the reference ``tilesynth`` package);
* :mod:`paper_2504_16214_b200.moe` -- the W4A16 MoE operator: sm_100a CUDA kernels
  (``csrc/``) behind the C ABI in ``include/w4a16_moe.h``.
"""
__version__ = "0.1.0"

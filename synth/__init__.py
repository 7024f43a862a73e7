"""Seeded synthetic KTH-shaped interest-point generator.

This module is shared by the oracle tests and the CUDA path.  It holds NONE of
the method's arithmetic (no model-graph selection, no scene sorting, no energy
terms): it only draws point sets.  Recipe: SURVEY.md §8(d) and DESIGN.md §3.

Paper facts used for the shapes:
  * frames of 160x120 pixels (§4),
  * F = 162 HoG/HoF components (§3.3),
  * lambda and T defaults and 60-frame blocks (§4),
  * 0-5 interest points per frame (§2.1).
"""
from .kth import (  # noqa: F401
    Points,
    Workload,
    FRAME_W,
    FRAME_H,
    F_KTH,
    gen_model,
    gen_clutter,
    make_recognition,
    make_single,
    RecognitionSet,
    gen_planted,
    concat_points,
    make_workload,
    CONFIGS,
)

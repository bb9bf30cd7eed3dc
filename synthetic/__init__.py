"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This package holds NO arithmetic of the BitStack method (no scaling, no sign
split, no SVD, no packing, no reconstruction).  It only draws random numbers
with the shapes and distributions of the paper's workloads (SURVEY.md §8(d),
"Synthetic inputs"), so that the oracle (oracle/) and the CUDA path
(paper_2410_23918_b200/) can be fed identical bytes while sharing no code.
"""
from .generators import (  # noqa: F401
    C4_LEVELS,
    CONFIGS,
    LLAMA31_8B_SHAPES,
    average_levels,
    seed_for,
    channel_gains,
    make_weight,
    make_calibration,
    make_x,
    make_random_blocks,
    random_signs_bytes,
)

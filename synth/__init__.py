"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the coding method's arithmetic (no window, MLP,
softmax, quantiser, rANS or schedule).  It only draws images and random
weights from fixed seeds, so both sides of every parity test see the same
bytes.  Recipes follow SURVEY.md §8(d) ("Concrete synthetic inputs"), which
shapes them after the paper's workloads: 8-bit grayscale photographs
(PAPER.md:37, P:110 CLIC 2019 mobile) and MRI slices whose colour frequencies
span ~1e4x (Fig. 5).
"""

from .images import (  # noqa: F401
    gradient_noise,
    natural_like,
    c2_image,
    mri_like_volume,
    mri_like_slices,
    random_image,
    config_images,
    CONFIGS,
)
from .weights import he_uniform_layers, he_uniform_pooled, zero_layers  # noqa: F401

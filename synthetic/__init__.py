"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the memory-layer method (no scoring, no
top-k, no softmax, no bag).  It only turns (seed, tag, counter) into numbers,
following the counter-based generator fixed in SURVEY.md §8(d):

    u_i = splitmix64(seed * 0x9E3779B97F4A7C15 + tag * 0xD1B54A32D192ED03 + i)

The CUDA library implements the same generator independently
(`ml_synth_fill` in paper_2412_09764_b200/csrc/synth.cu); a `-m gpu` test
checks the two bit for bit.  Because element (r, c) of an [R, C] tensor uses
counter i = r*C + c, any row of a huge table can be regenerated on demand,
so the oracle never needs a full 4-512 GiB value table in host memory.
"""
from .gen import (  # noqa: F401
    SEED_MUL, TAG_MUL, TAGS, CLS_CONTINUOUS, CLS_EXACT, CLS_DYADIC,
    splitmix64, counter_u64, unit_values, round_bf16, tensor, rows,
    bf16_bits, scale_for,
)
from .streams import (  # noqa: F401
    uniform_indices, zipf_indices, collision_indices, softmax_free_weights,
)

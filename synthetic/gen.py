"""Counter-based generator (SURVEY.md §8(d) "Synthetic inputs").

Classes of values (one per `cls`):

* CLS_CONTINUOUS: f = ((u >> 40) - 2^23) / 2^23 in [-1, 1) (24 significant
  bits, exact in fp32); value = fp32(f * scale) rounded to the dtype (RNE).
* CLS_EXACT:      f = (((u >> 60) & 15) - 8) / 8 in {-1, -7/8, ..., 7/8};
  exact in bf16; value = f * scale with scale a power of two (checked).
  Products of two such values are multiples of 1/64 and every sum the
  method forms from them stays exact in fp32 (SURVEY.md §8(c) pins).
* CLS_DYADIC:     f = ((u >> 58) & 63) / 64 in [0, 63/64]; used for bag
  weights in bit-exact bag tests.

All arithmetic is done in uint64 / fp32 exactly as the CUDA generator does it.
"""
import math

import numpy as np

SEED_MUL = 0x9E3779B97F4A7C15
TAG_MUL = 0xD1B54A32D192ED03
TAGS = {"q": 1, "K1": 2, "K2": 3, "V": 4, "x": 5, "W1": 6, "W2": 7,
        "dout": 8, "idx": 9, "w": 10}
CLS_CONTINUOUS, CLS_EXACT, CLS_DYADIC = 0, 1, 2

_M64 = (1 << 64) - 1


def splitmix64(x):
    """Standard splitmix64 output function applied to state x (uint64 array).

    splitmix64(0) == 0xE220A8397B1DCDAF (the published first output).
    """
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def counter_base(seed, tag):
    return (int(seed) * SEED_MUL + int(tag) * TAG_MUL) & _M64


def counter_u64(seed, tag, i):
    """u_i for an array of counters i (int64/uint64)."""
    base = np.uint64(counter_base(seed, tag))
    with np.errstate(over="ignore"):
        return splitmix64(base + np.asarray(i, dtype=np.uint64))


def round_bf16(x):
    """Round fp32 values to the nearest bf16 (ties to even); returns fp32."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    b = x.view(np.uint32).astype(np.uint64)
    lsb = (b >> np.uint64(16)) & np.uint64(1)
    b = ((b + np.uint64(0x7FFF) + lsb) & np.uint64(0xFFFF0000)).astype(np.uint32)
    return b.view(np.float32)


def bf16_bits(x):
    """uint16 bit patterns of bf16-representable fp32 values."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    return (x.view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def unit_values(u, cls):
    """Map u64 draws to fp32 unit values of the given class."""
    if cls == CLS_CONTINUOUS:
        m = (u >> np.uint64(40)).astype(np.int64) - (1 << 23)
        return m.astype(np.float32) * np.float32(1.0 / (1 << 23))
    if cls == CLS_EXACT:
        m = ((u >> np.uint64(60)) & np.uint64(15)).astype(np.int64) - 8
        return m.astype(np.float32) * np.float32(0.125)
    if cls == CLS_DYADIC:
        m = ((u >> np.uint64(58)) & np.uint64(63)).astype(np.int64)
        return m.astype(np.float32) * np.float32(1.0 / 64)
    raise ValueError(f"unknown class {cls}")


def _finish(f, scale, dtype, cls):
    if cls != CLS_CONTINUOUS:
        m, e = math.frexp(scale)
        if m != 0.5:
            raise ValueError("exact/dyadic classes need a power-of-two scale")
    v = (f * np.float32(scale)).astype(np.float32)
    if dtype == "bf16":
        v = round_bf16(v)
    elif dtype != "f32":
        raise ValueError(dtype)
    return v


def tensor(seed, tag, shape, scale=1.0, dtype="f32", cls=CLS_CONTINUOUS):
    """Whole tensor (fp32 array holding dtype-representable values)."""
    n = int(np.prod(shape))
    u = counter_u64(seed, TAGS.get(tag, tag), np.arange(n, dtype=np.uint64))
    return _finish(unit_values(u, cls), scale, dtype, cls).reshape(shape)


def rows(seed, tag, row_ids, ncols, scale=1.0, dtype="f32", cls=CLS_CONTINUOUS,
         col_lo=0, col_hi=None):
    """Rows `row_ids` (columns [col_lo, col_hi)) of an [R, ncols] tensor,
    regenerated on demand."""
    col_hi = ncols if col_hi is None else col_hi
    r = np.asarray(row_ids, dtype=np.uint64).reshape(-1, 1)
    c = np.arange(col_lo, col_hi, dtype=np.uint64).reshape(1, -1)
    with np.errstate(over="ignore"):
        i = r * np.uint64(ncols) + c
    u = counter_u64(seed, TAGS.get(tag, tag), i)
    return _finish(unit_values(u, cls), scale, dtype, cls)


def scale_for(tag, Dk=None, D=None, dv=None):
    """Scales of SURVEY.md §8(d): q, x, dout x1; K x 1/sqrt(Dk/2); V x1;
    W1 x 1/sqrt(D); W2 x 1/sqrt(dv). Returned as the fp32 constant both sides
    use (the CUDA generator receives it as an argument)."""
    if tag in ("K1", "K2"):
        return float(np.float32(1.0 / math.sqrt(Dk // 2)))
    if tag == "W1":
        return float(np.float32(1.0 / math.sqrt(D)))
    if tag == "W2":
        return float(np.float32(1.0 / math.sqrt(dv)))
    return 1.0

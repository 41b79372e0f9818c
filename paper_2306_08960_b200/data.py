"""Seeded synthetic operands in the reference's packed layouts (numpy, host side).

BASELINE.json's configs draw +-1 entries i.i.d. Bernoulli(0.5) and 2-bit codes
uniform over {0..3}. Uniform random uint64 words are exactly i.i.d. Bernoulli(0.5)
bits, so operands are generated as words directly (tail/padding bits masked to
zero, tensor.hpp:14-16). The reference's own generators (bench.cpp:37-55) use a
libstdc++ bernoulli stream; parity never depends on matching that stream because
both sides are handed the same words.
"""
from __future__ import annotations

import numpy as np

LANE_BITS = 512  # kDefaultLaneBits, tensor.hpp:17


def padded_words(cols: int, lane_bits: int = LANE_BITS) -> int:
    """tensor.cpp:21-27."""
    if lane_bits <= 0 or lane_bits % 64:
        raise ValueError("lane_bits must be a positive multiple of 64")
    if cols == 0:
        return 0
    return (cols + lane_bits - 1) // lane_bits * (lane_bits // 64)


def tail_mask_words(cols: int, wpr: int) -> np.ndarray:
    """Per-word keep masks for one row: ones for bits < cols, zeros in padding."""
    mask = np.zeros(wpr, dtype=np.uint64)
    full = cols // 64
    mask[:full] = np.uint64(0xFFFFFFFFFFFFFFFF)
    if cols % 64 and full < wpr:
        mask[full] = np.uint64((1 << (cols % 64)) - 1)
    return mask


def random_words(rng: np.random.Generator, rows: int, cols: int, lane_bits: int = LANE_BITS):
    """Uniform random bits in BitMatrix layout -> (words [rows, wpr] uint64, wpr)."""
    wpr = padded_words(cols, lane_bits)
    w = rng.integers(0, 2**64, size=(rows, wpr), dtype=np.uint64, endpoint=False)
    w &= tail_mask_words(cols, wpr)[None, :]
    return np.ascontiguousarray(w), wpr


def pack_bits(bits: np.ndarray, lane_bits: int = LANE_BITS):
    """0/1 array [rows, cols] -> (words [rows, wpr] uint64, wpr); bit i -> word i/64 bit i%64."""
    rows, cols = bits.shape
    wpr = padded_words(cols, lane_bits)
    padded = np.zeros((rows, wpr * 64), np.uint8)
    padded[:, :cols] = bits
    words = np.packbits(padded, axis=1, bitorder="little").view("<u8").reshape(rows, wpr)
    return np.ascontiguousarray(words.astype(np.uint64)), wpr


def unpack_bits(words: np.ndarray, cols: int) -> np.ndarray:
    """Inverse of pack_bits: [rows, wpr] uint64 -> 0/1 uint8 [rows, cols]."""
    rows = words.shape[0]
    b = np.unpackbits(np.ascontiguousarray(words).view(np.uint8).reshape(rows, -1), axis=1,
                      bitorder="little")
    return b[:, :cols]


def random_levels(rng: np.random.Generator, rows: int, cols: int) -> np.ndarray:
    return rng.integers(0, 4, size=(rows, cols), dtype=np.uint8)


def planes_from_levels(levels: np.ndarray, lane_bits: int = LANE_BITS):
    """decompose_thm table (transform.cpp:47-75): p0->(0,0,1) p1->(0,0,0) p2->(0,1,0) p3->(1,0,1).
    Returns (t, h, m, wpr)."""
    t, wpr = pack_bits((levels == 3).astype(np.uint8), lane_bits)
    h, _ = pack_bits((levels == 2).astype(np.uint8), lane_bits)
    m, _ = pack_bits(((levels == 0) | (levels == 3)).astype(np.uint8), lane_bits)
    return t, h, m, wpr


def random_planes(rng: np.random.Generator, rows: int, cols: int, lane_bits: int = LANE_BITS):
    """Uniform 2-bit codes in {t,h,m} plane form, generated word-parallel (fast at 32k x 32k).
    Returns (t, h, m, wpr)."""
    b1, wpr = random_words(rng, rows, cols, lane_bits)  # level bit 1
    b0, _ = random_words(rng, rows, cols, lane_bits)    # level bit 0
    keep = tail_mask_words(cols, wpr)[None, :]
    t = b1 & b0             # level 3
    h = b1 & ~b0 & keep     # level 2
    m = (~b1 & ~b0 & keep) | t  # level 0 or 3
    return np.ascontiguousarray(t), np.ascontiguousarray(h), np.ascontiguousarray(m), wpr


def levels_from_planes(t: np.ndarray, h: np.ndarray, m: np.ndarray, cols: int) -> np.ndarray:
    """recompose_thm (transform.cpp:77-96) on legal planes."""
    tb, hb, mb = unpack_bits(t, cols), unpack_bits(h, cols), unpack_bits(m, cols)
    return np.where(mb == 1, np.where(tb == 1, 3, 0), np.where(hb == 1, 2, 1)).astype(np.uint8)


def apb_weights(rng: np.random.Generator, out_features: int, in_features: int,
                std: float = 0.02, keep_frac: float = 0.02):
    """BASELINE config 4 weights: w ~ N(0, std); per output row alpha_r = mean|w_r|; the top
    `keep_frac` |w| entries of each row stay full precision, every other entry becomes
    alpha_r * sign(w) — i.e. the output of apb_forward (apb.cpp:57-68) with a per-row
    threshold. Returns (a [rows, cols] fp32 forward output, alpha [rows] fp32, kept count/row)."""
    w = rng.normal(0.0, std, size=(out_features, in_features)).astype(np.float32)
    alpha = np.abs(w).mean(axis=1, dtype=np.float64).astype(np.float32)
    keep = max(1, int(round(keep_frac * in_features)))
    order = np.argsort(-np.abs(w), axis=1, kind="stable")
    keep_mask = np.zeros_like(w, dtype=bool)
    np.put_along_axis(keep_mask, order[:, :keep], True, axis=1)
    sign = np.where(w >= 0.0, np.float32(1.0), np.float32(-1.0))
    a = np.where(keep_mask, w, sign * alpha[:, None]).astype(np.float32)
    return a, alpha, keep

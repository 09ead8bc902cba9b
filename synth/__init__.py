"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no products, no sums over k):
it only draws the input matrices A, B, C_in from a counter-based generator so
that any row, shard or sampled sub-block can be regenerated without the whole
matrix ("Inputs").

Generator ("Input recipe"):
    key  = seed * 2^40  XOR  matrix_id * 2^56  XOR  (i * cols + j)
    u    = splitmix64(key) >> 40                      (24 uniform bits)
    v    = u * 2^-23 - 1                              (uniform on [-1, 1), exact in f32)
    A, B, F16 C_in: v rounded to binary16 (RNE, numpy's cast)
    F32 C_in:      v as float32 (exact)
Matrix ids: A = 0, B = 1, C = 2.  The distribution (uniform [-1, 1]) follows the
SPEC's reading of the paper's unspecified test data (seeds 0-4
S:518); the paper itself is silent (reading R14).
"""
from __future__ import annotations

import numpy as np

MATRIX_A = 0
MATRIX_B = 1
MATRIX_C = 2

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 finaliser on uint64 (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = x + _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def uniform_f32(seed: int, matrix_id: int, rows: int, cols: int,
                row_ids=None, col_lo: int = 0, col_hi: int | None = None) -> np.ndarray:
    """Uniform [-1,1) float32 values of the logical rows x cols matrix.

    row_ids / [col_lo, col_hi) select a sub-block (same values as in the full
    matrix).  Values are exactly representable in float32.
    """
    if not (0 <= seed < 2 ** 16):
        raise ValueError("seed must be in [0, 2^16)")
    if rows * cols >= 2 ** 40:
        raise ValueError("matrix too large for the key packing")
    if col_hi is None:
        col_hi = cols
    r = np.arange(rows, dtype=np.uint64) if row_ids is None else np.asarray(row_ids, dtype=np.uint64)
    c = np.arange(col_lo, col_hi, dtype=np.uint64)
    base = (np.uint64(seed) << np.uint64(40)) ^ (np.uint64(matrix_id) << np.uint64(56))
    out = np.empty((r.shape[0], c.shape[0]), dtype=np.float32)
    # chunk rows to bound temporaries (~64 MB of uint64 per chunk)
    step = max(1, (1 << 23) // max(1, c.shape[0]))
    for s in range(0, r.shape[0], step):
        rr = r[s:s + step]
        idx = rr[:, None] * np.uint64(cols) + c[None, :]
        u = splitmix64(base ^ idx) >> np.uint64(40)
        out[s:s + step] = (u.astype(np.float32) * np.float32(2.0 ** -23)) - np.float32(1.0)
    return out


def uniform_f16(seed: int, matrix_id: int, rows: int, cols: int, **kw) -> np.ndarray:
    """uniform_f32 rounded to binary16 (round-to-nearest-even)."""
    return uniform_f32(seed, matrix_id, rows, cols, **kw).astype(np.float16)


def to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """float32 -> bfloat16 bit patterns (uint16), round to nearest even (NaN kept quiet)."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    with np.errstate(over="ignore"):
        r = (b + np.uint32(0x7FFF) + ((b >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)
    nan = (b & np.uint32(0x7FFFFFFF)) > np.uint32(0x7F800000)
    r = np.where(nan, (b >> np.uint32(16)) | np.uint32(0x40), r)
    return r.astype(np.uint16)


def uniform_bf16(seed: int, matrix_id: int, rows: int, cols: int, **kw) -> np.ndarray:
    """uniform_f32 rounded to bfloat16, returned as uint16 bit patterns."""
    return to_bf16_bits(uniform_f32(seed, matrix_id, rows, cols, **kw))


def problem(M: int, N: int, K: int, acc: str = "f32", seed: int = 0):
    """(A (M,K) f16, B (K,N) f16, C_in (M,N) f32|f16) for one seeded problem."""
    A = uniform_f16(seed, MATRIX_A, M, K)
    B = uniform_f16(seed, MATRIX_B, K, N)
    if acc == "f32":
        C = uniform_f32(seed, MATRIX_C, M, N)
    elif acc == "f16":
        C = uniform_f16(seed, MATRIX_C, M, N)
    else:
        raise ValueError(acc)
    return A, B, C


def problem_bf16(M: int, N: int, K: int, acc: str = "f32", seed: int = 0):
    """(A bf16 bits (M,K) uint16, B bf16 bits (K,N) uint16, C_in f32|f16) -- BF16 inputs."""
    A = uniform_bf16(seed, MATRIX_A, M, K)
    B = uniform_bf16(seed, MATRIX_B, K, N)
    C = uniform_f32(seed, MATRIX_C, M, N) if acc == "f32" else uniform_f16(seed, MATRIX_C, M, N)
    return A, B, C


def sample_rows(M: int, tile_m: int = 128, n_random: int = 64, seed: int = 0) -> np.ndarray:
    """Rows for sampled parity at full size: first/last row of every tile row-block
    boundary region plus seeded random rows."""
    rng = np.random.default_rng(1000 + seed)
    rows = set()
    for t in range(0, M, tile_m):
        rows.add(t)
        rows.add(min(M - 1, t + tile_m - 1))
    rows.update(int(x) for x in rng.integers(0, M, size=n_random))
    return np.array(sorted(rows), dtype=np.int64)

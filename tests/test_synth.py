"""The seeded input generator (synth/): determinism, sub-block consistency, range."""
import numpy as np

import synth


def test_splitmix64_known_vector():
    # splitmix64 with state 0: first output of the reference generator (Steele et al.)
    assert int(synth.splitmix64(np.array([0], dtype=np.uint64))[0]) == 0xE220A8397B1DCDAF


def test_deterministic_and_subblocks_match():
    full = synth.uniform_f32(3, synth.MATRIX_A, 50, 70)
    again = synth.uniform_f32(3, synth.MATRIX_A, 50, 70)
    assert np.array_equal(full, again)
    rows = [0, 7, 49]
    sub = synth.uniform_f32(3, synth.MATRIX_A, 50, 70, row_ids=rows, col_lo=10, col_hi=33)
    assert np.array_equal(sub, full[rows, 10:33])
    other = synth.uniform_f32(4, synth.MATRIX_A, 50, 70)
    assert not np.array_equal(full, other)
    assert not np.array_equal(full, synth.uniform_f32(3, synth.MATRIX_B, 50, 70))


def test_range_and_grid():
    v = synth.uniform_f32(0, 0, 300, 300)
    assert v.min() >= -1.0 and v.max() < 1.0
    assert abs(float(v.mean())) < 0.01
    # every value is on the 2^-23 grid: (v + 1) * 2^23 is an integer
    q = (v.astype(np.float64) + 1.0) * 2.0 ** 23
    assert np.array_equal(q, np.round(q))
    h = synth.uniform_f16(0, 0, 300, 300)
    assert h.dtype == np.float16 and np.array_equal(h, v.astype(np.float16))


def test_sample_rows_cover_tile_edges():
    rows = synth.sample_rows(1000, tile_m=128, n_random=5)
    for t in range(0, 1000, 128):
        assert t in rows and min(999, t + 127) in rows
    assert rows.min() >= 0 and rows.max() < 1000


def test_bf16_rounding_matches_torch():
    import torch
    rng = np.random.default_rng(3)
    x = np.concatenate([rng.standard_normal(20000).astype(np.float32) * np.float32(10.0) ** rng.integers(-30, 30, 20000).astype(np.float32),
                        np.array([0.0, -0.0, 1.0, 65504.0, 3.0e38, np.inf, -np.inf, 1e-40], np.float32)])
    ours = synth.to_bf16_bits(x)
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(ours, ref)

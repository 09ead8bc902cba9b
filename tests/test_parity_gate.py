"""CPU pins of the parity gate itself (tests/parity.py): the F16 element-wise bound accepts
the correctly rounded result and rejects the localized failures the Frobenius bar alone
misses (a 256 x 512 tile that dropped its C_in passes 2e-3)."""
import numpy as np
import pytest

import oracle
import synth
from parity import check, f16_element_bound, ulp16


def test_ulp16_closed_forms():
    assert ulp16(1.0) == 2.0 ** -10 and ulp16(1.5) == 2.0 ** -10 and ulp16(2.0) == 2.0 ** -9
    assert ulp16(65504.0) == 32.0 and ulp16(-3.0) == 2.0 ** -9
    assert ulp16(0.0) == 2.0 ** -24 and ulp16(2.0 ** -20) == 2.0 ** -24 and ulp16(2.0 ** -14) == 2.0 ** -24


def _problem(M=96, N=600, K=1024):
    A, B, C = synth.problem(M, N, K, "f16", seed=3)
    ex, rnd = oracle.gemm(A, B, C)
    return A, B, C, ex, rnd


def test_gate_accepts_the_correctly_rounded_result():
    A, B, C, ex, rnd = _problem()
    s = check(rnd, ex, A, B, "f16", A.shape[1], "RNE of the exact result")
    assert s["elem_slack_min"] > 0


def test_gate_rejects_a_tile_that_dropped_c_in():
    A, B, C, ex, rnd = _problem(M=512, N=1024, K=4096)
    bad = rnd.copy()
    # one 16-row x 128-column block (1/256 of C) computed as A.B without its C_in:
    # rel-Frobenius stays below 2e-3, but every element with |C_in| above the bound is caught
    blk = (slice(32, 48), slice(256, 384))
    bad[blk] = (ex[blk] - C[blk].astype(np.float64)).astype(np.float16)
    rel = np.linalg.norm(bad.astype(np.float64) - ex) / np.linalg.norm(ex)
    assert rel < 2e-3
    with pytest.raises(AssertionError, match="element bound"):
        check(bad, ex, A, B, "f16", A.shape[1], "dropped C_in")


def test_gate_rejects_a_few_ulps_error_on_one_element():
    A, B, C, ex, rnd = _problem()
    bound = f16_element_bound(ex, A, B, A.shape[1])
    i = (5, 77)
    bad = rnd.copy()
    bad[i] = np.float16(ex[i] + 1.5 * bound[i] * np.sign(ex[i] or 1.0))
    with pytest.raises(AssertionError, match="element bound"):
        check(bad, ex, A, B, "f16", A.shape[1], "one element off")


def test_extra_roundings_widen_only_by_half_an_ulp_of_s_each():
    A, B, C, ex, rnd = _problem(M=8, N=16, K=64)
    b0 = f16_element_bound(ex, A, B, 64)
    b2 = f16_element_bound(ex, A, B, 64, extra_roundings=2)
    S = (np.abs(A.astype(np.float32)) @ np.abs(B.astype(np.float32))).astype(np.float64) * 1.01
    assert np.allclose(b2 - b0, ulp16(S))

"""Pins for the CPU oracle (oracle/oracle.c) against things other than itself.

Each pin is chosen so a plausible mistake in the oracle fails at least one:
  - a wrong binary16 decode/encode      -> all-65536-pattern decode, numpy encode
  - a dropped C_in term / wrong sign    -> hand fixture, A=0 / B=0 closed forms
  - a transposed or mis-indexed operand -> permutation, rank-1, exact rationals
  - a wrong lda/ldb/ldc stride          -> padded-ld equality
  - a wrong rounding of the output      -> exact rationals + numpy RNE casts
Citations: PAPER.md P:908-909 (C = AB + C, row-major), P:412-438 (naive loop),
P:926-930 (F16 in, F32 acc/out), P:976-980 (F16 in/acc/out).
"""
import json
import math
import os
import subprocess
import sys
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def _f16(x):
    return np.asarray(x, dtype=np.float16)


# ---------------------------------------------------------------- binary16 codec

def test_f16_decoder_all_patterns():
    bits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    ref = bits.view(np.float16).astype(np.float64)
    got = np.array([oracle.f16_to_f64(int(b)) for b in bits])
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(got), nan)
    assert np.array_equal(got[~nan], ref[~nan])
    # signed zeros keep their sign
    assert math.copysign(1.0, oracle.f16_to_f64(0x8000)) == -1.0


def _np_f16_bits(x):
    import warnings
    warnings.simplefilter("ignore", RuntimeWarning)
    return int(np.array([x], dtype=np.float64).astype(np.float16).view(np.uint16)[0])


def test_f16_encoder_matches_numpy_rne():
    rng = np.random.default_rng(0)
    vals = list(rng.standard_normal(4000) * 10.0 ** rng.uniform(-9, 5.5, 4000))
    # ties and boundaries: halfway between representable neighbours
    for h in range(0, 0x7c00, 37):
        lo = np.uint16(h).view(np.float16).astype(np.float64)
        hi = np.uint16(h + 1).view(np.float16).astype(np.float64)
        vals += [lo, (lo + hi) / 2, np.nextafter((lo + hi) / 2, 0), np.nextafter((lo + hi) / 2, 1e9)]
    vals += [65504.0, 65519.99, 65520.0, 70000.0, 2.0 ** -24, 2.0 ** -25, 3 * 2.0 ** -26,
             2.0 ** -25 + 2.0 ** -40, 2.0 ** -14, 2.0 ** -14 - 2.0 ** -25, 1e-30, 0.0, -0.0,
             float("inf"), -float("inf")]
    vals += [-v for v in vals]
    for v in vals:
        assert oracle.f64_to_f16_bits(v) == _np_f16_bits(v), v
    assert oracle.f64_to_f16_bits(float("nan")) & 0x7c00 == 0x7c00
    assert oracle.f64_to_f16_bits(float("nan")) & 0x3ff != 0


# ---------------------------------------------------------------- fixtures / exact

def test_hand_worked_fixture():
    with open(os.path.join(HERE, "golden", "hand_2x3x2.json")) as f:
        g = json.load(f)
    A = _f16(g["A"])
    B = _f16(g["B"])
    for acc, dt in ((oracle.ACC_F32, np.float32), (oracle.ACC_F16, np.float16)):
        C = np.asarray(g["C_in"], dtype=dt)
        ex, rd = oracle.gemm(A, B, C, acc)
        assert np.array_equal(ex, np.asarray(g["C_out"], dtype=np.float64))
        assert np.array_equal(rd.astype(np.float64), np.asarray(g["C_out"], dtype=np.float64))


def _exact(A, B, C, i, j):
    s = Fraction(float(C[i, j]))
    for k in range(A.shape[1]):
        s += Fraction(float(A[i, k])) * Fraction(float(B[k, j]))
    return s


@pytest.mark.parametrize("acc", ["f32", "f16"])
def test_exact_rationals_tiny_shapes(acc):
    rng = np.random.default_rng(1)
    u = 2.0 ** -53
    for trial in range(40):
        M, N, K = (int(x) for x in rng.integers(1, 14, size=3))
        if trial < 3:
            K = 1
        A, B, C = synth.problem(M, N, K, acc, seed=trial % 5)
        # widen the dynamic range so additions actually round in double
        A = (A.astype(np.float32) * np.float32(2.0) ** rng.integers(-12, 8, size=A.shape)).astype(np.float16)
        ex, rd = oracle.gemm(A, B, C)
        gamma = (K + 1) * u / (1 - (K + 1) * u)
        for i in range(M):
            for j in range(N):
                e = _exact(A, B, C, i, j)
                bound = gamma * (abs(float(C[i, j])) + sum(abs(float(A[i, k]) * float(B[k, j])) for k in range(K)))
                assert abs(Fraction(ex[i, j]) - e) <= Fraction(bound), (M, N, K, i, j)
        # one RNE rounding of the double result to the output type
        want = ex.astype(np.float32) if acc == "f32" else ex.astype(np.float16)
        assert np.array_equal(rd.view(np.uint8), want.view(np.uint8))


def test_numpy_float64_256_cube():
    for acc in ("f32", "f16"):
        A, B, C = synth.problem(256, 256, 256, acc, seed=3)
        ex, rd = oracle.gemm(A, B, C)
        ref = A.astype(np.float64) @ B.astype(np.float64) + C.astype(np.float64)
        K = 256
        gamma = (K + 1) * 2.0 ** -53 / (1 - (K + 1) * 2.0 ** -53)
        bound = 2 * gamma * (np.abs(A.astype(np.float64)) @ np.abs(B.astype(np.float64)) + np.abs(C.astype(np.float64)))
        assert np.all(np.abs(ex - ref) <= bound)


# ---------------------------------------------------------------- closed forms

@pytest.mark.parametrize("acc", ["f32", "f16"])
def test_identity_gives_B(acc):
    K, N = 96, 77
    _, B, C = synth.problem(K, N, K, acc, seed=0)
    A = np.eye(K, dtype=np.float16)
    C0 = np.zeros((K, N), dtype=C.dtype)
    ex, rd = oracle.gemm(A, B, C0)
    assert np.array_equal(ex, B.astype(np.float64))
    assert np.array_equal(rd.astype(np.float64), B.astype(np.float64))


def test_permutation_permutes_rows():
    K, N = 64, 40
    _, B, _ = synth.problem(K, N, K, "f32", seed=1)
    perm = np.random.default_rng(5).permutation(K)
    P = np.zeros((K, K), dtype=np.float16)
    P[np.arange(K), perm] = 1
    ex, _ = oracle.gemm(P, B, np.zeros((K, N), np.float32))
    assert np.array_equal(ex, B.astype(np.float64)[perm])


@pytest.mark.parametrize("acc", ["f32", "f16"])
def test_zero_operand_leaves_C_bitwise(acc):
    A, B, C = synth.problem(33, 45, 70, acc, seed=2)
    for AA, BB in ((np.zeros_like(A), B), (A, np.zeros_like(B))):
        _, rd = oracle.gemm(AA, BB, C)
        assert np.array_equal(rd.view(np.uint8), C.view(np.uint8))


def test_K_zero_leaves_C():
    _, _, C = synth.problem(5, 6, 1, "f32", seed=0)
    _, rd = oracle.gemm(np.zeros((5, 0), np.float16), np.zeros((0, 6), np.float16), C)
    assert np.array_equal(rd, C)


@pytest.mark.parametrize("K,acc", [(1, "f32"), (1000, "f32"), (4096, "f32"), (2048, "f16"), (777, "f16")])
def test_all_ones_gives_K(K, acc):
    M, N = 9, 11
    A = np.ones((M, K), np.float16)
    B = np.ones((K, N), np.float16)
    C = np.zeros((M, N), np.float32 if acc == "f32" else np.float16)
    ex, rd = oracle.gemm(A, B, C)
    assert np.all(ex == K) and np.all(rd.astype(np.float64) == K)


def test_rank1_powers_of_two():
    M, N, K = 12, 10, 48
    a = np.arange(M) % 7
    b = np.arange(N) % 5
    A = np.repeat((2.0 ** -a)[:, None], K, axis=1).astype(np.float16)
    B = np.repeat((2.0 ** -b)[None, :], K, axis=0).astype(np.float16)
    ex, rd = oracle.gemm(A, B, np.zeros((M, N), np.float32))
    want = K * 2.0 ** -(a[:, None] + b[None, :])
    assert np.array_equal(ex, want) and np.array_equal(rd.astype(np.float64), want)


def test_small_integers_exact_vs_integer_matmul():
    rng = np.random.default_rng(7)
    M, N, K = 70, 50, 300
    Ai = rng.integers(-2, 3, size=(M, K))
    Bi = rng.integers(-2, 3, size=(K, N))
    Ci = rng.integers(-100, 101, size=(M, N))
    ex, rd = oracle.gemm(Ai.astype(np.float16), Bi.astype(np.float16), Ci.astype(np.float32))
    want = (Ai @ Bi + Ci).astype(np.float64)  # integer arithmetic, exact
    assert np.array_equal(ex, want) and np.array_equal(rd.astype(np.float64), want)


def test_subnormal_product():
    A = np.array([[2.0 ** -24]], np.float16)
    B = np.array([[1.0]], np.float16)
    ex, rd = oracle.gemm(A, B, np.zeros((1, 1), np.float32))
    assert ex[0, 0] == 2.0 ** -24 and rd[0, 0] == np.float32(2.0 ** -24)


def test_special_values_propagate():
    A, B, C = synth.problem(4, 5, 6, "f16", seed=0)
    A = A.copy()
    A[1, 2] = np.float16("nan")
    A[2, 0] = np.float16("inf")
    B = np.abs(B) + np.float16(0.5)
    _, rd = oracle.gemm(A, B, C)
    assert np.all(np.isnan(rd[1]))
    assert np.all(np.isposinf(rd[2]))
    # overflow of the F16 output rounds to Inf (no saturation, R5)
    big = np.full((1, 1), 60000.0, np.float16)
    _, rd = oracle.gemm(np.full((1, 4), 64.0, np.float16), np.full((4, 1), 64.0, np.float16), big)
    assert np.isposinf(rd[0, 0])


# ---------------------------------------------------------------- layout / rows

def test_padded_leading_dims_and_row_subset():
    M, N, K = 37, 29, 51
    A, B, C = synth.problem(M, N, K, "f32", seed=4)
    ex, rd = oracle.gemm(A, B, C)
    Ap = np.full((M, K + 13), np.float16("nan"))
    Ap[:, :K] = A
    Bp = np.full((K, N + 3), np.float16("nan"))
    Bp[:, :N] = B
    Cp = np.full((M, N + 7), np.float32("nan"))
    Cp[:, :N] = C
    ex2, rd2 = oracle.gemm(Ap[:, :K], Bp[:, :N], Cp[:, :N])
    assert np.array_equal(ex, ex2)
    rows = [0, 5, 36, 17]
    ex3, rd3 = oracle.gemm(A, B, C, rows=rows)
    assert np.array_equal(ex3, ex[rows]) and np.array_equal(rd3, rd[rows])


def test_thread_count_independent():
    code = ("import sys; sys.path.insert(0, %r); import numpy as np, oracle, synth;"
            "A,B,C = synth.problem(200,150,300,'f32',seed=1);"
            "ex,_ = oracle.gemm(A,B,C); sys.stdout.write(ex.tobytes().hex()[:4000] + str(hash(ex.tobytes())))") % ROOT
    outs = []
    for t in ("1", "5"):
        env = dict(os.environ, OMP_NUM_THREADS=t, PYTHONHASHSEED="0")
        outs.append(subprocess.run([sys.executable, "-c", code], env=env, capture_output=True,
                                   text=True, check=True).stdout)
    assert outs[0] == outs[1]


def test_invalid_arguments_rejected():
    A, B, C = synth.problem(4, 4, 4, "f32")
    with pytest.raises(ValueError):
        oracle.gemm(A, B, C, rows=[4])
    with pytest.raises(ValueError):
        oracle.gemm(A, B[:3], C)


# ---------------------------------------------------------------- NEXT #4 extensions
# (BF16 inputs P:272-275, fused bias / ReLU P:87-89, beta = 0)

def test_bf16_decoder_all_patterns():
    import torch
    bits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    ref = torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16).to(torch.float64).numpy()
    got = np.array([oracle.bf16_to_f64(int(b)) for b in bits])
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(got), nan)
    assert np.array_equal(got[~nan], ref[~nan])


def _bf16_val(bits):
    import torch
    return torch.from_numpy(np.asarray(bits).view(np.int16)).view(torch.bfloat16).to(torch.float64).numpy()


def test_bf16_exact_rationals():
    rng = np.random.default_rng(8)
    for trial in range(20):
        M, N, K = (int(x) for x in rng.integers(1, 12, size=3))
        A, B, C = synth.problem_bf16(M, N, K, "f32", seed=trial % 5)
        ex, _ = oracle.gemm(A, B, C, in_type=1)
        Av, Bv = _bf16_val(A), _bf16_val(B)
        u = 2.0 ** -53
        gamma = (K + 1) * u / (1 - (K + 1) * u)
        for i in range(M):
            for j in range(N):
                e = Fraction(float(C[i, j])) + sum(Fraction(float(Av[i, k])) * Fraction(float(Bv[k, j])) for k in range(K))
                bound = gamma * (abs(float(C[i, j])) + sum(abs(Av[i, k] * Bv[k, j]) for k in range(K)))
                assert abs(Fraction(ex[i, j]) - e) <= Fraction(bound)


def test_beta0_ignores_C_in():
    K, N = 80, 56
    _, B, _ = synth.problem(K, N, K, "f32", seed=2)
    C_nan = np.full((K, N), np.nan, np.float32)
    ex, rd = oracle.gemm(np.eye(K, dtype=np.float16), B, C_nan, beta=0)
    assert np.array_equal(ex, B.astype(np.float64)) and np.array_equal(rd, B.astype(np.float32))


def test_bias_broadcast_and_relu_closed_forms():
    rng = np.random.default_rng(9)
    M, N, K = 40, 33, 70
    Ai = rng.integers(-2, 3, size=(M, K))
    Bi = rng.integers(-2, 3, size=(K, N))
    Ci = rng.integers(-60, 61, size=(M, N))
    bias = rng.integers(-30, 31, size=N).astype(np.float32)
    for relu in (False, True):
        for beta in (0, 1):
            ex, rd = oracle.gemm(Ai.astype(np.float16), Bi.astype(np.float16), Ci.astype(np.float32),
                                 beta=beta, bias=bias, relu=relu)
            want = (Ai @ Bi + beta * Ci + bias.astype(np.int64)[None, :]).astype(np.float64)
            if relu:
                want = np.maximum(want, 0.0)
            assert np.array_equal(ex, want), (relu, beta)
    # A = 0: out = relu(C_in + bias), per column
    A0 = np.zeros((M, K), np.float16)
    ex, _ = oracle.gemm(A0, Bi.astype(np.float16), Ci.astype(np.float32), bias=bias, relu=True)
    assert np.array_equal(ex, np.maximum(Ci + bias[None, :].astype(np.int64), 0).astype(np.float64))


def test_relu_keeps_nan():
    A = np.array([[np.nan, 1.0]], np.float16)
    B = np.array([[1.0], [1.0]], np.float16)
    ex, rd = oracle.gemm(A, B, np.zeros((1, 1), np.float32), relu=True)
    assert np.isnan(ex[0, 0]) and np.isnan(rd[0, 0])
    ex, _ = oracle.gemm(np.array([[-3.0]], np.float16), np.array([[2.0]], np.float16), np.zeros((1, 1), np.float32), relu=True)
    assert ex[0, 0] == 0.0

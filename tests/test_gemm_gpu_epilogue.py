"""GPU parity for the fused-epilogue extension: BF16 inputs,
beta = 0, per-column bias, ReLU -- against the oracle's oracle_gemm_ex, which
follows the same definition:  C <- relu?(beta * C_in + A.B + bias[j])."""
import itertools

import numpy as np
import pytest

import oracle
import synth
from parity import check, round_up

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    import paper_2108_13191_b200 as g
    g.load_library()
    return g


def _dev(host, pad=8, dtype=None):
    """Device copy with a padded leading dimension (16-byte multiple) as a view."""
    import torch
    t = torch.from_numpy(np.ascontiguousarray(host))
    if dtype is not None:
        t = t.view(dtype)
    ld = round_up(host.shape[1] + pad, 8)
    full = torch.zeros((host.shape[0], ld), dtype=t.dtype)
    full[:, : host.shape[1]] = t
    return full.cuda()[:, : host.shape[1]]


CASES = list(itertools.product(["f16", "bf16"], [1, 0], [False, True], [False, True]))


@pytest.mark.parametrize("in_t,beta,use_bias,relu", CASES)
@pytest.mark.parametrize("acc", ["f32", "f16"])
def test_fused_epilogue_parity(g, in_t, beta, use_bias, relu, acc):
    import torch
    M, N, K = 520, 708, 777          # ragged tiles; N*2 % 16 != 0 for F16 C -> masked store path too
    if in_t == "bf16":
        A, B, C = synth.problem_bf16(M, N, K, acc, seed=50)
        dA, dB = _dev(A, dtype=torch.bfloat16), _dev(B, dtype=torch.bfloat16)
    else:
        A, B, C = synth.problem(M, N, K, acc, seed=50)
        dA, dB = _dev(A), _dev(B)
    bias = synth.uniform_f32(51, 3, 1, N)[0] * np.float32(4.0) if use_bias else None
    dbias = torch.from_numpy(bias).cuda() if use_bias else None
    for cfg in ("auto", "pair_256x256_k128", "solo_128x64", "pair_256x256_s5"):
        dC = _dev(C)
        g.gemm_f16(dA, dB, dC, config=cfg, beta=beta, bias=dbias, relu=relu)
        torch.cuda.synchronize()
        ex, _ = oracle.gemm(A, B, C, in_type=1 if in_t == "bf16" else 0, beta=beta, bias=bias, relu=relu)
        Av = A if in_t == "f16" else torch.from_numpy(A.view(np.int16)).view(torch.bfloat16).float().numpy()
        Bv = B if in_t == "f16" else torch.from_numpy(B.view(np.int16)).view(torch.bfloat16).float().numpy()
        check(dC.cpu().numpy(), ex, Av, Bv, acc, K, f"{in_t} beta={beta} bias={use_bias} relu={relu} {acc} {cfg}")
        if relu:
            assert (dC.cpu().numpy() >= 0).all()


def test_fused_epilogue_closed_forms(g):
    """Exact cases: small integers (F32 exact), beta = 0 with a NaN-filled C (never
    read), bias only (A = 0), ReLU clamps negatives to +0 and keeps NaN."""
    import torch
    rng = np.random.default_rng(12)
    M, N, K = 300, 264, 400
    Ai = rng.integers(-2, 3, size=(M, K))
    Bi = rng.integers(-2, 3, size=(K, N))
    Ci = rng.integers(-40, 41, size=(M, N))
    bias = rng.integers(-20, 21, size=N).astype(np.float32)
    dA, dB, db = _dev(Ai.astype(np.float16)), _dev(Bi.astype(np.float16)), torch.from_numpy(bias).cuda()
    for beta, relu in itertools.product((1, 0), (False, True)):
        dC = _dev(Ci.astype(np.float32)) if beta else _dev(np.full((M, N), np.nan, np.float32))
        g.gemm_f16(dA, dB, dC, beta=beta, bias=db, relu=relu)
        want = Ai @ Bi + beta * Ci + bias.astype(np.int64)[None, :]
        if relu:
            want = np.maximum(want, 0)
        assert np.array_equal(dC.cpu().numpy(), want.astype(np.float32)), (beta, relu)
    # NaN in A propagates through ReLU
    An = Ai.astype(np.float16)
    An[3, 7] = np.float16("nan")
    dC = _dev(Ci.astype(np.float32))
    g.gemm_f16(_dev(An), dB, dC, relu=True)
    out = dC.cpu().numpy()
    assert np.isnan(out[3]).all() and not np.isnan(np.delete(out, 3, axis=0)).any()


def test_fused_epilogue_argument_errors(g):
    import torch
    A = torch.zeros((64, 64), dtype=torch.float16, device="cuda")
    B = torch.zeros((64, 64), dtype=torch.bfloat16, device="cuda")
    C = torch.zeros((64, 64), dtype=torch.float32, device="cuda")
    with pytest.raises(TypeError):
        g.gemm_f16(A, B, C)                      # mixed input types
    with pytest.raises(ValueError):
        g.gemm_f16(A, A, C, bias=torch.zeros(63, device="cuda"))
    with pytest.raises(ValueError):
        g.gemm_f16(A, A, C, beta=2)
    misaligned = torch.zeros(65, device="cuda")[1:]
    with pytest.raises(g.GemmError) as e:
        g.gemm_f16(A, A, C, bias=misaligned)
    assert e.value.status == 2

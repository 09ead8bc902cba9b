"""GPU parity for the split-K cluster kernels (csrc/gemm_sm100_splitk.cuh:
GEMM_CFG_SPLITK_128x256_S2 / _S4, SPLITK_128x128_S4) against the CPU oracle.

What is new in them: S CTAs of a cluster accumulate disjoint K ranges, the partials
meet in distributed shared memory, and each CTA reduces, adds C_in and stores its
column slice with plain (vector or element-wise) global accesses.  The cases aim
at the K partition (K shorter than S k-blocks, so some CTAs hold an empty share;
ragged K), the column-slice ownership (ragged N, odd N), guard bands, a grid of
more clusters than fit at once, and the fixed reduction order (bitwise
determinism).  Bars as everywhere: BASELINE.json north_star (tests/parity.py)."""
import itertools

import numpy as np
import pytest

import oracle
import synth
from parity import Guarded, check, device_problem, oracle_full, round_up

pytestmark = pytest.mark.gpu

SPLIT = ["splitk_128x256_s2", "splitk_128x256_s4", "splitk_128x128_s4", "splitk_128x128_s2"]


@pytest.fixture(scope="module")
def g():
    import torch
    import paper_2108_13191_b200 as g
    assert torch.cuda.is_available()
    g.load_library()
    return g


def _run(g, gA, gB, gC, cfg, **kw):
    import torch
    g.gemm_f16(gA.view, gB.view, gC.view, config=cfg, **kw)
    torch.cuda.synchronize()


@pytest.mark.parametrize("cfg", SPLIT)
@pytest.mark.parametrize("acc", ["f32", "f16"])
@pytest.mark.parametrize("shape", [(601, 712, 333), (128, 256, 64), (129, 257, 1000), (1, 1, 1), (300, 9, 17),
                                   (257, 515, 129), (1024, 1024, 1024)])
def test_splitk_ragged_guarded(g, cfg, acc, shape):
    M, N, K = shape
    A, B, C, gA, gB, gC = device_problem(M, N, K, acc, seed=M + N, pad=(8, 16, 8))
    _run(g, gA, gB, gC, cfg)
    ex, _ = oracle_full(A, B, C)
    check(gC.result(), ex, A, B, acc, K, f"{cfg} {acc} {shape}")
    assert gC.guard_intact(), "write outside the M x N window"


@pytest.mark.parametrize("cfg", SPLIT)
def test_splitk_empty_shares(g, cfg):
    # K = 64 or 100: one or two k-blocks for up to 4 CTAs -- the others contribute zero
    for K in (8, 64, 100, 192):
        for acc in ("f32", "f16"):
            A, B, C, gA, gB, gC = device_problem(200, 300, K, acc, seed=K)
            _run(g, gA, gB, gC, cfg)
            ex, _ = oracle_full(A, B, C)
            check(gC.result(), ex, A, B, acc, K, f"{cfg} K={K} {acc}")


@pytest.mark.parametrize("cfg", SPLIT)
def test_splitk_closed_forms_bit_exact(g, cfg):
    # all ones: C = K exactly; small integers exact in F32 whatever the split
    for K in (16, 1000, 2048):
        gA = Guarded(np.ones((130, K), np.float16), K)
        gB = Guarded(np.ones((K, 200), np.float16), 200)
        gC = Guarded(np.zeros((130, 200), np.float32), 200)
        _run(g, gA, gB, gC, cfg)
        assert np.all(gC.result() == K), K
    rng = np.random.default_rng(31)
    M, N, K = 260, 392, 700
    Ai = rng.integers(-2, 3, size=(M, K))
    Bi = rng.integers(-2, 3, size=(K, N))
    Ci = rng.integers(-50, 51, size=(M, N))
    gA = Guarded(Ai.astype(np.float16), round_up(K, 8))
    gB = Guarded(Bi.astype(np.float16), N)
    gC = Guarded(Ci.astype(np.float32), N)
    _run(g, gA, gB, gC, cfg)
    assert np.array_equal(gC.result().astype(np.int64), Ai @ Bi + Ci)
    # A = 0 leaves C bitwise unchanged (every partial is +0)
    A, B, C, gA, gB, gC = device_problem(200, 136, 96, "f16", seed=4)
    gA.full.zero_()
    _run(g, gA, gB, gC, cfg)
    assert np.array_equal(gC.result().view(np.uint8), C.view(np.uint8))


@pytest.mark.parametrize("cfg", SPLIT)
def test_splitk_many_waves_and_determinism(g, cfg):
    # more clusters than fit on the GPU at once (non-persistent grid), run twice: bitwise equal
    import torch
    M, N, K = 2048, 2048, 512
    A, B, C, gA, gB, gC = device_problem(M, N, K, "f32", seed=9)
    outs = []
    for _ in range(2):
        gC.full.copy_(torch.from_numpy(gC.full_host.copy()))
        _run(g, gA, gB, gC, cfg)
        outs.append(gC.result().copy())
    assert np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32))
    rows = synth.sample_rows(M, tile_m=128, n_random=8, seed=9)
    ex, _ = oracle.gemm(A, B, C, rows=rows)
    check(outs[0][rows], ex, A[rows], B, "f32", K, f"{cfg} many waves")


CASES = list(itertools.product(["f16", "bf16"], [1, 0], [False, True], [False, True]))


@pytest.mark.parametrize("in_t,beta,use_bias,relu", CASES)
@pytest.mark.parametrize("acc", ["f32", "f16"])
def test_splitk_fused_epilogue(g, in_t, beta, use_bias, relu, acc):
    import torch
    M, N, K = 300, 530, 777
    def dev(host, dtype=None):
        # device copy with a leading dimension padded to a 16-byte multiple, as a view
        t = torch.from_numpy(np.ascontiguousarray(host))
        if dtype is not None:
            t = t.view(dtype)
        full = torch.zeros((host.shape[0], round_up(host.shape[1], 8) + 8), dtype=t.dtype)
        full[:, : host.shape[1]] = t
        return full.cuda()[:, : host.shape[1]]

    if in_t == "bf16":
        A, B, C = synth.problem_bf16(M, N, K, acc, seed=60)
        dA, dB = dev(A.view(np.int16), torch.bfloat16), dev(B.view(np.int16), torch.bfloat16)
    else:
        A, B, C = synth.problem(M, N, K, acc, seed=60)
        dA, dB = dev(A), dev(B)
    bias = synth.uniform_f32(61, 3, 1, N)[0] * np.float32(4.0) if use_bias else None
    dbias = torch.from_numpy(bias).cuda() if use_bias else None
    Av = A if in_t == "f16" else torch.from_numpy(A.view(np.int16)).view(torch.bfloat16).float().numpy()
    Bv = B if in_t == "f16" else torch.from_numpy(B.view(np.int16)).view(torch.bfloat16).float().numpy()
    ex, _ = oracle.gemm(A, B, C, in_type=1 if in_t == "bf16" else 0, beta=beta, bias=bias, relu=relu)
    for cfg in SPLIT:
        dC = dev(C)
        g.gemm_f16(dA, dB, dC, config=cfg, beta=beta, bias=dbias, relu=relu)
        torch.cuda.synchronize()
        check(dC.cpu().numpy(), ex, Av, Bv, acc, K, f"{cfg} {in_t} beta={beta} bias={use_bias} relu={relu} {acc}")


def test_splitk_rejects_promotion(g):
    import torch
    A = torch.zeros((128, 64), dtype=torch.float16, device="cuda")
    B = torch.zeros((64, 256), dtype=torch.float16, device="cuda")
    C = torch.zeros((128, 256), dtype=torch.float32, device="cuda")
    with pytest.raises(g.GemmError):
        g.gemm_f16(A, B, C, config="splitk_128x256_s4", promote_k=512)
    info = g.config_info("splitk_128x256_s4", g.ACC_F32)
    assert info["tile_m"] == 128 and info["tile_n"] == 256 and info["cta_group"] == 1


@pytest.mark.parametrize("shape", [(256, 512, 16384), (512, 512, 8192), (1024, 1024, 8192), (128, 4096, 4096)])
def test_splitk_auto_long_k_accuracy(g, shape):
    # the shapes pick_config sends to a split-K config; F32 C keeps each CTA's TMEM
    # chain <= 4096 long (R4), so the error stays well under the 1e-5 bar
    import torch
    M, N, K = shape
    assert g.pick_config(M, N, K, g.ACC_F32) in (10, 11, 12, 15)
    assert g.pick_config(M, N, K, g.ACC_F16) in (10, 11, 12, 15)
    for acc in ("f32", "f16"):
        A, B, C = synth.problem(M, N, K, acc, seed=11)
        dA, dB, dC = (torch.from_numpy(x).cuda() for x in (A, B, C))
        g.gemm_f16(dA, dB, dC)
        torch.cuda.synchronize()
        rows = synth.sample_rows(M, tile_m=128, n_random=8, seed=11)
        ex, _ = oracle.gemm(A, B, C, rows=rows)
        s = check(dC[torch.from_numpy(rows).cuda()].cpu().numpy(), ex, A[rows], B, acc, K, f"auto {shape} {acc}")
        if acc == "f32":
            assert s["rel_fro"] < 6e-6, s

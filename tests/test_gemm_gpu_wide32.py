"""GPU parity for the 256 x 512 CTA-pair tile with F32 C (csrc/gemm_sm100_wide_f32.cuh,
GEMM_CFG_PAIR_256x512 with GEMM_ACC_F32) against the CPU oracle.

What is new in this kernel, and what the cases aim at:
  * K-chunk promotion by TMA reduce-add into C, at staggered points for the two accumulator
    halves (h0 after Cb, 2 Cb, ... k-blocks, h1 after Cb/2, 3 Cb/2, ...): every k-block must
    land in C exactly once (integer-exact cases with many promotion points), in a fixed
    order (bitwise repeatable, independent of the grid);
  * the MMA issuer's run-ahead on one half while the other drains (deferred MMAs, stage
    release once both halves used a stage), at every ring depth;
  * the tile-tail hand-over (h0 first) and the head of the next tile (phase wrap);
  * beta = 0 (first drain stores) and bias (added once) in the EXT build; the F32 bars of
    BASELINE.json north_star, long-K accuracy (chains <= promote_k + a few k-blocks).
PAPER.md P:908-909 (C = AB + C), Sec. 4.1 P:924-949 (F32 accumulate)."""
import numpy as np
import pytest

import oracle
import synth
from parity import Guarded, check, device_problem, oracle_full, round_up, stats

pytestmark = pytest.mark.gpu

W = "pair_256x512"


@pytest.fixture(scope="module")
def g():
    import torch
    import paper_2108_13191_b200 as g
    assert torch.cuda.is_available()
    g.load_library()
    return g


def _run(g, gA, gB, gC, **kw):
    import torch
    g.gemm_f16(gA.view, gB.view, gC.view, config=W, **kw)
    torch.cuda.synchronize()


@pytest.mark.parametrize("shape", [(601, 1100, 333), (256, 512, 64), (257, 516, 65), (1, 4, 1), (1000, 1032, 1000),
                                   (512, 2048, 1536), (300, 8, 40), (130, 700, 2100), (700, 1300, 5000)])
@pytest.mark.parametrize("promote_k", [0, -1, 768])
def test_wide32_ragged_guarded(g, shape, promote_k):
    M, N, K = shape
    A, B, C, gA, gB, gC = device_problem(M, N, K, "f32", seed=7, pad=(8, 16, 8))
    _run(g, gA, gB, gC, promote_k=promote_k)
    ex, _ = oracle_full(A, B, C)
    check(gC.result(), ex, A, B, "f32", K, f"{W} f32 {shape} promote_k={promote_k}")
    assert gC.guard_intact(), "write outside the M x N window"
    assert gA.guard_intact() and gB.guard_intact()


@pytest.mark.parametrize("promote_k", [768, 1024, 1536, 4096, -1])
@pytest.mark.parametrize("ring_stages", [0, 1, 2, 3])
def test_wide32_every_k_block_once_exact(g, promote_k, ring_stages):
    # integer A, B in {-2..2}, C_in integers: every partial sum is an integer < 2^24, exact in
    # F32 in any order -- a k-block that is skipped, doubled or drained twice changes the result
    rng = np.random.default_rng(promote_k & 0xFFFF)
    M, N, K = 520, 1040, 4800
    Ai = rng.integers(-2, 3, size=(M, K))
    Bi = rng.integers(-2, 3, size=(K, N))
    Ci = rng.integers(-1000, 1001, size=(M, N))
    gA = Guarded(Ai.astype(np.float16), round_up(K, 8))
    gB = Guarded(Bi.astype(np.float16), N)
    gC = Guarded(Ci.astype(np.float32), N)
    _run(g, gA, gB, gC, promote_k=promote_k, ring_stages=ring_stages)
    assert np.array_equal(gC.result().astype(np.int64), Ai @ Bi + Ci)
    assert gC.guard_intact()


def test_wide32_rejects_promotion_points_too_close(g):
    import torch
    A = torch.zeros((256, 4096), dtype=torch.float16, device="cuda")
    B = torch.zeros((4096, 512), dtype=torch.float16, device="cuda")
    C = torch.zeros((256, 512), dtype=torch.float32, device="cuda")
    with pytest.raises(g.GemmError):          # Cb = 8 k-blocks: Cb / 2 < ring_stages + 2
        g.gemm_f16(A, B, C, config=W, promote_k=512)
    g.gemm_f16(A, B, C, config=W, promote_k=512, ring_stages=2)   # Cb / 2 = 4 >= 2 + 2
    with pytest.raises(g.GemmError):          # ReLU is not built for F32 C on this tile
        g.gemm_f16(A, B, C, config=W, relu=True)
    Cr = torch.zeros((256, 512), dtype=torch.float32, device="cuda")[:, :510]
    with pytest.raises(g.GemmError):          # N * 4 % 16 != 0: reduce-add would overrun
        g.gemm_f16(A, B[:, :510], Cr, config=W)


@pytest.mark.parametrize("max_clusters", [1, 3])
def test_wide32_persistent_phase_wrap(g, max_clusters):
    M, N, K = 1300, 2100, 2000
    A, B, C, gA, gB, gC = device_problem(M, N, K, "f32", seed=3)
    _run(g, gA, gB, gC, max_clusters=max_clusters, promote_k=768)
    ex, _ = oracle_full(A, B, C)
    check(gC.result(), ex, A, B, "f32", K, f"{W} clusters={max_clusters}")


def test_wide32_deterministic_and_schedule_independent(g):
    import torch
    M, N, K = 1024, 2048, 4096
    A, B, C, gA, gB, gC = device_problem(M, N, K, "f32", seed=6)
    outs = []
    for mc in (0, 0, 3, 1):
        gC.full.copy_(torch.from_numpy(gC.full_host.copy()))
        _run(g, gA, gB, gC, max_clusters=mc, promote_k=1024)
        outs.append(gC.result().view(np.uint32).copy())
    for o in outs[1:]:
        assert np.array_equal(outs[0], o)


@pytest.mark.parametrize("beta", [1, 0])
@pytest.mark.parametrize("use_bias", [False, True])
@pytest.mark.parametrize("in_t", ["f16", "bf16"])
def test_wide32_fused_epilogue(g, beta, use_bias, in_t):
    import torch
    M, N, K = 520, 1104, 2000   # (row pitches of A, B and C multiples of 16 bytes: TMA)
    if in_t == "bf16":
        A, B, C = synth.problem_bf16(M, N, K, "f32", seed=50)
        dA = torch.from_numpy(A.view(np.int16)).view(torch.bfloat16).cuda()
        dB = torch.from_numpy(B.view(np.int16)).view(torch.bfloat16).cuda()
        Av = dA.float().cpu().numpy()
        Bv = dB.float().cpu().numpy()
    else:
        A, B, C = synth.problem(M, N, K, "f32", seed=50)
        dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
        Av, Bv = A, B
    bias = synth.uniform_f32(51, 3, 1, N)[0] * np.float32(4.0) if use_bias else None
    dC = torch.from_numpy(C.copy()).cuda()
    g.gemm_f16(dA, dB, dC, config=W, beta=beta, bias=None if bias is None else torch.from_numpy(bias).cuda(),
               promote_k=768)
    torch.cuda.synchronize()
    ex, _ = oracle.gemm(A, B, C, in_type=1 if in_t == "bf16" else 0, beta=beta, bias=bias)
    check(dC.cpu().numpy(), ex, Av, Bv, "f32", K, f"{W} f32 {in_t} beta={beta} bias={use_bias}")


def test_wide32_long_k_accuracy(g):
    # K = 16384: chains of <= 4096 (+ guard) k, promoted by RN reduce-adds -- the error stays
    # near the chain length's, not K's (single chain: ~2e-5, over the 1e-5 bar)
    import torch
    M, N, K = 256, 1024, 16384
    A, B, C = synth.problem(M, N, K, "f32", seed=9)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    ex, _ = oracle.gemm(A, B, C)
    rel = {}
    for pk in (0, -1):
        dC = torch.from_numpy(C.copy()).cuda()
        g.gemm_f16(dA, dB, dC, config=W, promote_k=pk)
        torch.cuda.synchronize()
        rel[pk] = stats(dC.cpu().numpy(), ex)["rel_fro"]
        if pk == 0:
            check(dC.cpu().numpy(), ex, A, B, "f32", K, "wide32 K=16384")
    print(f"wide32 K=16384 rel_fro: promoted {rel[0]:.3e}, single chain {rel[-1]:.3e}")
    assert rel[0] <= 7e-6 < rel[-1]


def test_wide32_8192_cube_sampled(g):
    import torch
    M = N = K = 8192
    A, B, C = synth.problem(M, N, K, "f32", seed=0)
    dA, dB, dC = (torch.from_numpy(x).cuda() for x in (A, B, C))
    g.gemm_f16(dA, dB, dC, config=W)
    torch.cuda.synchronize()
    rows = synth.sample_rows(M, tile_m=256, n_random=8)[::4]
    got = dC[torch.from_numpy(rows).cuda()].cpu().numpy()
    ex, _ = oracle.gemm(A, B, C, rows=rows)
    s = check(got, ex, A[rows], B, "f32", K, "8192^3 wide32 sampled")
    print(f"8192^3 wide32: rel_fro {s['rel_fro']:.3e}")

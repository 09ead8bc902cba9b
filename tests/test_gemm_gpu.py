"""GPU parity: the CUDA path (libgemm_f16.so through the Python binding over the C ABI)
against the CPU oracle, element by element on the same seeded inputs.

Bars (BASELINE.json north_star, restated in tests/parity.py): F32 accumulate
max|err| <= 1e-3 sqrt(K) max|A| max|B| and rel-Frobenius <= 1e-5; F16
rel-Frobenius <= 2e-3.  Closed forms are bit-exact.  PAPER.md P:908-909.
"""
import numpy as np
import pytest

import oracle
import synth
from parity import Guarded, check, device_problem, oracle_full, round_up, stats

pytestmark = pytest.mark.gpu

CFGS = ["pair_256x256", "pair_256x128", "solo_128x256", "solo_128x128", "solo_128x64", "solo_128x64_mc4",
        "solo_128x128_mc4"]


@pytest.fixture(scope="module")
def g():
    import torch
    import paper_2108_13191_b200 as g
    assert torch.cuda.is_available()
    g.load_library()
    return g


def _run(g, gA, gB, gC, **kw):
    import torch
    g.gemm_f16(gA.view, gB.view, gC.view, **kw)
    torch.cuda.synchronize()


@pytest.mark.parametrize("acc", ["f32", "f16"])
def test_smoke_256_cube(g, acc):
    M = N = K = 256
    A, B, C, gA, gB, gC = device_problem(M, N, K, acc, seed=0)
    _run(g, gA, gB, gC)
    ex, _ = oracle_full(A, B, C)
    check(gC.result(), ex, A, B, acc, K, "256^3 auto")
    assert gC.guard_intact()


@pytest.mark.parametrize("cfg", CFGS)
@pytest.mark.parametrize("acc", ["f32", "f16"])
def test_configs_ragged_multi_tile(g, cfg, acc):
    # several tiles in M and N, ragged M/N/K tails, padded leading dims
    M, N, K = 601, 712, 333
    A, B, C, gA, gB, gC = device_problem(M, N, K, acc, seed=1, pad=(8, 16, 8))
    _run(g, gA, gB, gC, config=cfg)
    ex, _ = oracle_full(A, B, C)
    check(gC.result(), ex, A, B, acc, K, f"{cfg} {acc}")
    assert gC.guard_intact(), "write outside the M x N window"
    assert gA.guard_intact() and gB.guard_intact()


@pytest.mark.parametrize("cfg", CFGS)
def test_persistent_loop_phase_wrap(g, cfg):
    # one cluster walks every tile: exercises ring/TMEM phase bits across many tiles
    M, N, K = 1100, 900, 640
    A, B, C, gA, gB, gC = device_problem(M, N, K, "f32", seed=2)
    _run(g, gA, gB, gC, config=cfg, max_clusters=1)
    ex, _ = oracle_full(A, B, C)
    check(gC.result(), ex, A, B, "f32", K, f"{cfg} one cluster")


@pytest.mark.parametrize("acc", ["f32", "f16"])
def test_closed_forms_bit_exact(g, acc):
    import torch
    # identity: A = I (M = K), C_in = 0 -> C = B exactly
    K, N = 384, 320
    B = synth.uniform_f16(3, 1, K, N)
    dt = np.float32 if acc == "f32" else np.float16
    gA = Guarded(np.eye(K, dtype=np.float16), K)
    gB = Guarded(B, N)
    gC = Guarded(np.zeros((K, N), dt), N)
    _run(g, gA, gB, gC)
    assert np.array_equal(gC.result().astype(np.float64), B.astype(np.float64))
    # all ones: C = K (F32 exact for any K <= 2^24; F16 exact for K <= 2048)
    for K in (16, 1000, 2048):
        M, N = 130, 200
        gA = Guarded(np.ones((M, K), np.float16), K)
        gB = Guarded(np.ones((K, N), np.float16), N)
        gC = Guarded(np.zeros((M, N), dt), N)
        _run(g, gA, gB, gC)
        assert np.all(gC.result() == K), K
    # A = 0 leaves C bitwise unchanged
    A, Bm, C, gA, gB, gC = device_problem(200, 136, 96, acc, seed=4)
    gA.full.zero_()
    _run(g, gA, gB, gC)
    assert np.array_equal(gC.result().view(np.uint8), C.view(np.uint8))


def test_small_integers_exact_f32(g):
    rng = np.random.default_rng(11)
    M, N, K = 520, 392, 700
    Ai = rng.integers(-2, 3, size=(M, K))
    Bi = rng.integers(-2, 3, size=(K, N))
    Ci = rng.integers(-50, 51, size=(M, N))
    gA = Guarded(Ai.astype(np.float16), round_up(K, 8))
    gB = Guarded(Bi.astype(np.float16), N)
    gC = Guarded(Ci.astype(np.float32), N)
    for cfg in CFGS:
        gC.full.copy_(__import__("torch").from_numpy(gC.full_host.copy()))
        _run(g, gA, gB, gC, config=cfg)
        assert np.array_equal(gC.result().astype(np.int64), Ai @ Bi + Ci), cfg


def test_permutation_rows(g):
    K, N = 256, 264
    perm = np.random.default_rng(9).permutation(K)
    P = np.zeros((K, K), np.float16)
    P[np.arange(K), perm] = 1
    B = synth.uniform_f16(0, 1, K, N)
    gA, gB, gC = Guarded(P, K), Guarded(B, N), Guarded(np.zeros((K, N), np.float32), N)
    _run(g, gA, gB, gC, config="pair_256x256")
    assert np.array_equal(gC.result(), B.astype(np.float32)[perm])


@pytest.mark.parametrize("acc", ["f32", "f16"])
def test_brute_force_tiny_shapes(g, acc):
    rng = np.random.default_rng(5)
    shapes = [(1, 1, 1), (1, 8, 1), (7, 9, 15), (33, 40, 17), (40, 1, 40), (2, 3, 64), (17, 24, 65)]
    shapes += [tuple(int(x) for x in rng.integers(1, 41, size=3)) for _ in range(12)]
    for (M, N, K) in shapes:
        A, B, C, gA, gB, gC = device_problem(M, N, K, acc, seed=M + N + K, pad=(8, 8, 8))
        _run(g, gA, gB, gC)
        ex, _ = oracle_full(A, B, C)
        check(gC.result(), ex, A, B, acc, K, f"{(M, N, K)}")
        assert gC.guard_intact(), (M, N, K)


def test_deterministic_and_schedule_independent(g):
    import torch
    M, N, K = 1024, 768, 512
    A, B, C, gA, gB, gC = device_problem(M, N, K, "f32", seed=6)
    outs = []
    for mc in (0, 0, 3):
        gC.full.copy_(torch.from_numpy(gC.full_host.copy()))
        _run(g, gA, gB, gC, config="pair_256x256", max_clusters=mc)
        outs.append(gC.result().copy())
    assert np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32))
    assert np.array_equal(outs[0].view(np.uint32), outs[2].view(np.uint32))


def test_rounding_probe_reports(g, capsys):
    """P4: k16 block 0 contributes 1, block 1 contributes 3*2^-25.
    RNE accumulation gives 1 + 2^-23, truncation gives 1.  Reported, and the F32
    tolerance must hold either way."""
    K = 32
    A = np.zeros((128, K), np.float16)
    B = np.zeros((K, 128), np.float16)
    A[0, 0] = 1.0
    B[0, 0] = 1.0
    for k in (16, 17, 18):
        A[0, k] = 2.0 ** -12
        B[k, 0] = 2.0 ** -13
    gA, gB, gC = Guarded(A, K), Guarded(B, 128), Guarded(np.zeros((128, 128), np.float32), 128)
    _run(g, gA, gB, gC)
    v = float(gC.result()[0, 0])
    mode = "RNE-like" if v == 1.0 + 2.0 ** -23 else ("truncating" if v == 1.0 else f"other ({v!r})")
    print(f"F32 accumulate rounding probe: {mode}")
    assert v in (1.0, 1.0 + 2.0 ** -23)


@pytest.mark.parametrize("acc", ["f32", "f16"])
def test_host_buffer_e2e_path(g, acc):
    import torch
    M, N, K = 300, 264, 200
    A, B, C = synth.problem(M, N, K, acc, seed=8)
    hA = torch.from_numpy(A).pin_memory()
    hB = torch.from_numpy(B).pin_memory()
    hC = torch.from_numpy(C.copy()).pin_memory()
    dA = torch.empty((M, round_up(K, 8)), dtype=torch.float16, device="cuda")[:, :K]
    dB = torch.empty((K, N), dtype=torch.float16, device="cuda")
    dC = torch.empty((M, N), dtype=hC.dtype, device="cuda")
    g.gemm_f16_host(hA, hB, hC, dA, dB, dC)
    torch.cuda.synchronize()
    ex, _ = oracle_full(A, B, C)
    check(hC.numpy(), ex, A, B, acc, K, "host path")


def test_errors_are_reported(g):
    import torch
    A = torch.zeros((64, 64), dtype=torch.float16, device="cuda")
    B = torch.zeros((64, 64), dtype=torch.float16, device="cuda")
    C = torch.zeros((64, 64), dtype=torch.float32, device="cuda")
    big = torch.zeros(64 * 64 + 8, dtype=torch.float16, device="cuda")
    misA = big[1:1 + 64 * 64].view(64, 64)
    with pytest.raises(g.GemmError) as e:
        g.gemm_f16(misA, B, C)
    assert e.value.status == 2
    with pytest.raises(g.GemmError) as e:
        g.gemm_f16(A, B, C, config=99)
    assert e.value.status == 1
    # K == 0: nothing launched, C unchanged
    C0 = C.clone()
    g.gemm_f16(A[:, :0], B[:0, :], C)
    assert g.last_launches() == 0 and torch.equal(C, C0)


@pytest.mark.parametrize("promote_k", [64, 128, 512, 2048, -1])
@pytest.mark.parametrize("cfg", ["pair_256x256", "solo_128x64"])
def test_promotion_chunk_lengths(g, promote_k, cfg):
    """K chunks of every length (incl. one chunk per k-block and a ragged last
    chunk) give oracle parity; -1 = one TMEM chain per tile."""
    M, N, K = 600, 712, 1000
    A, B, C, gA, gB, gC = device_problem(M, N, K, "f32", seed=12)
    _run(g, gA, gB, gC, config=cfg, promote_k=promote_k)
    ex, _ = oracle_full(A, B, C)
    check(gC.result(), ex, A, B, "f32", K, f"promote_k={promote_k}")


def test_promotion_bounds_long_k_error(g):
    """DESIGN.md R4: a single TMEM chain truncates, so its error grows with K and
    fails the 1e-5 bound at K=16384; chunked promotion (default) keeps it small."""
    import torch
    M, N, K = 256, 512, 16384
    A, B, C = synth.problem(M, N, K, "f32", seed=2)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    ex, _ = oracle.gemm(A, B, C)
    rel = {}
    for pk in (0, -1):
        dC = torch.from_numpy(C.copy()).cuda()
        g.gemm_f16(dA, dB, dC, promote_k=pk, config="pair_256x256")   # (auto would split K here)
        torch.cuda.synchronize()
        rel[pk] = stats(dC.cpu().numpy(), ex)["rel_fro"]
    print(f"K=16384 rel_fro: promoted {rel[0]:.3e}, single chain {rel[-1]:.3e}")
    assert rel[0] <= 5e-6 < rel[-1]


@pytest.mark.parametrize("kw", [
    {"ring_stages": 1}, {"ring_stages": 2}, {"acc_bufs": 1}, {"acc_bufs": 1, "ring_stages": 1},
    {"group_m": 1}, {"group_m": 3}, {"raster": 1}, {"raster": 1, "group_m": 2}, {"c_reduce": 1}, {"c_reduce": -1},
    {"c_reduce": 1, "config": "pair_256x256_s5"}, {"c_reduce": 1, "config": "solo_128x64"}, {"l2_hints": -1},
    {"max_clusters": 1000},
    {"config": "pair_256x256_s5"}, {"config": "pair_256x256_s4"}, {"config": "solo_128x256", "ring_stages": 1, "acc_bufs": 1},
    {"pdl": -1}, {"tail_ring": -1}, {"stream_k": -1}, {"l2_hints": 1, "group_m": 16},
    {"swizzle": -1}, {"swizzle": -1, "ring_stages": 1}, {"swizzle": -1, "promote_k": 256},
    {"warp_specialize": -1}, {"warp_specialize": -1, "ring_stages": 1}, {"warp_specialize": -1, "promote_k": 512},
])
def test_ablation_knobs_keep_parity(g, kw):
    """Every ablation switch (used by tools/ablation.py) is a scheduling choice only:
    results stay within the bar (and a 1-deep ring stresses the phase logic)."""
    M, N, K = 777, 1040, 1216
    for acc in ("f32", "f16"):
        A, B, C, gA, gB, gC = device_problem(M, N, K, acc, seed=13)
        _run(g, gA, gB, gC, **kw)
        ex, _ = oracle_full(A, B, C)
        check(gC.result(), ex, A, B, acc, K, f"{kw} {acc}")
        assert gC.guard_intact()


@pytest.mark.parametrize("M", [1, 1000, 2300, 9000])
def test_host_path_row_block_pipeline(g, M):
    """gemm_f16_host splits M into row blocks (H2D / GEMM / D2H on three streams):
    every block, including a ragged last one, matches the oracle."""
    import torch
    N, K = 264, 136
    for acc in ("f32", "f16"):
        A, B, C = synth.problem(M, N, K, acc, seed=M)
        hA = torch.from_numpy(A).pin_memory()
        hB = torch.from_numpy(B).pin_memory()
        hC = torch.from_numpy(C.copy()).pin_memory()
        dA = torch.empty((M, K), dtype=torch.float16, device="cuda")
        dB = torch.empty((K, N), dtype=torch.float16, device="cuda")
        dC = torch.empty((M, N), dtype=hC.dtype, device="cuda")
        s = torch.cuda.Stream()
        g.gemm_f16_host(hA, hB, hC, dA, dB, dC, stream=s)
        s.synchronize()
        ex, _ = oracle_full(A, B, C)
        check(hC.numpy(), ex, A, B, acc, K, f"host pipeline M={M}")


@pytest.mark.parametrize("M", [700, 3000])
def test_host_path_resident_operands(g, M):
    """gemm_f16_host with hA/hB = None reuses A/B already in dA/dB (the bench's e2e
    step: one F32 and one F16 GEMM on the same operands copy A and B once); dA/dB
    are poisoned before the first call so a missed copy cannot pass."""
    import torch
    N, K = 520, 264
    A, B, C32 = synth.problem(M, N, K, "f32", seed=M + 1)
    _, _, C16 = synth.problem(M, N, K, "f16", seed=M + 1)
    hA = torch.from_numpy(A).pin_memory()
    hB = torch.from_numpy(B).pin_memory()
    hC32 = torch.from_numpy(C32.copy()).pin_memory()
    hC16 = torch.from_numpy(C16.copy()).pin_memory()
    dA = torch.full((M, K), float("nan"), dtype=torch.float16, device="cuda")
    dB = torch.full((K, N), float("nan"), dtype=torch.float16, device="cuda")
    dC32 = torch.empty((M, N), dtype=torch.float32, device="cuda")
    dC16 = torch.empty((M, N), dtype=torch.float16, device="cuda")
    s = torch.cuda.Stream()
    g.gemm_f16_host(hA, hB, hC32, dA, dB, dC32, stream=s)
    g.gemm_f16_host(None, None, hC16, dA, dB, dC16, stream=s)
    s.synchronize()
    check(hC32.numpy(), oracle_full(A, B, C32)[0], A, B, "f32", K, "host, A/B copied")
    check(hC16.numpy(), oracle_full(A, B, C16)[0], A, B, "f16", K, "host, A/B resident")
    # only B resident: a new A is copied, the old B reused
    A2 = synth.uniform_f16(M + 7, 0, M, K)
    hC16b = torch.from_numpy(C16.copy()).pin_memory()
    g.gemm_f16_host(torch.from_numpy(A2).pin_memory(), None, hC16b, dA, dB, dC16, stream=s)
    s.synchronize()
    check(hC16b.numpy(), oracle_full(A2, B, C16)[0], A2, B, "f16", K, "host, B resident")


@pytest.mark.parametrize("cfg", ["solo_128x64_mc4", "solo_128x128_mc4"])
@pytest.mark.parametrize("acc", ["f32", "f16"])
@pytest.mark.parametrize("shape", [(1024, 1024, 1024), (130, 70, 200), (300, 1000, 777), (129, 640, 64), (1, 1, 1)])
def test_a_multicast_configs(g, cfg, acc, shape):
    """4-CTA clusters share A by TMA multicast: each CTA loads a quarter of the A box
    for all four.  Cases: N tiles not a multiple of 4 (CTAs whose tile lies wholly
    outside C still load their quarter of A and must write nothing), one cluster
    walking all tiles (phase wrap), ragged K, guard bands."""
    M, N, K = shape
    A, B, C, gA, gB, gC = device_problem(M, N, K, acc, seed=M + K, pad=(8, 8, 8))
    for mc in (0, 1):
        gC.full.copy_(__import__("torch").from_numpy(gC.full_host.copy()))
        _run(g, gA, gB, gC, config=cfg, max_clusters=mc)
        ex, _ = oracle_full(A, B, C)
        check(gC.result(), ex, A, B, acc, K, f"{cfg} {acc} {shape} clusters={mc}")
        assert gC.guard_intact(), "write outside the M x N window"


@pytest.mark.parametrize("cfg", ["pair_256x256_s5", "pair_256x256_k128", "pair_256x256", "solo_128x64",
                                 "solo_128x64_mc4"])
def test_c_reduce_bitwise_equal_to_staged(g, cfg):
    """F32 C by TMA reduce-add (c_reduce): the L2 adds the staged accumulator into C_in
    -- the same single IEEE RN add as the staged path, so the results must be bitwise
    equal, on a ragged, padded, guard-banded problem whose C_in holds -0.0, +-Inf, NaN
    and subnormals too."""
    import torch
    M, N, K = 777, 1000, 1000                      # N % 4 == 0: reduce-add applies
    A, B, C, gA, gB, gC = device_problem(M, N, K, "f32", seed=13, pad=(8, 8, 4))
    C = C.copy()
    C[::7, ::5] = -0.0
    C[3, :8] = [np.inf, -np.inf, np.nan, 1e-40, -1e-40, 3.4e38, -3.4e38, 0.0]
    base = Guarded(C, gC.ld)
    outs = []
    for red in (1, -1):
        gC.full.copy_(torch.from_numpy(base.full_host.copy()))
        _run(g, gA, gB, gC, config=cfg, c_reduce=red)
        outs.append(gC.result().copy())
        assert gC.guard_intact()
    assert np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32))
    finite = np.isfinite(C).all(axis=1)
    ex, _ = oracle_full(A, B, C)
    check(outs[0][finite], ex[finite], A[finite], B, "f32", K, f"c_reduce {cfg}")


def test_pdl_mixed_kernel_chain_exact(g):
    """The bench's launch pattern under PDL: different kernels back to back on one stream
    (F32 pair tile with the reduce-add epilogue, F16 256x512 tile, split-K, 1-CTA), each
    reading what an earlier one wrote, so every kernel's prologue overlaps a different
    kernel's tail.  Small-integer inputs make every result exact."""
    import torch
    rng = np.random.default_rng(17)
    M, N, K = 512, 1024, 2048
    A = torch.from_numpy(rng.integers(-1, 2, (M, K)).astype(np.float16)).cuda()
    B = torch.from_numpy(rng.integers(-1, 2, (K, N)).astype(np.float16)).cuda()
    C32 = torch.from_numpy(rng.integers(-40, 41, (M, N)).astype(np.float32)).cuda()
    C16 = torch.from_numpy(rng.integers(-40, 41, (M, N)).astype(np.float16)).cuda()
    AB = (A.double() @ B.double())
    want32 = C32.double().clone()
    want16 = C16.double().clone()
    seq = [("f32", "pair_256x256_k128"), ("f16", "pair_256x512"), ("f32", "splitk_128x128_s4"),
           ("f16", "pair_256x512"), ("f32", "solo_128x64"), ("f16", "splitk_128x256_s2"), ("f32", "pair_256x256")]
    for _ in range(2):
        for mode, cfg in seq:
            if mode == "f32":
                g.gemm_f16(A, B, C32, config=cfg, pdl=1)
                want32 += AB
            else:
                g.gemm_f16(A, B, C16, config=cfg, pdl=1)
                want16 += AB
    torch.cuda.synchronize()
    assert float(want16.abs().max()) <= 2048          # every F16 result exact
    assert torch.equal(C32.double(), want32)
    assert torch.equal(C16.double(), want16)


def test_cuda_graph_capture_replay(g):
    """The C ABI is capturable: gemm_f16 calls recorded into a CUDA graph replay
    to the same results as eager calls (tensor maps travel as kernel params)."""
    import torch
    M, N, K = 640, 520, 384
    A, B, C = synth.problem(M, N, K, "f32", seed=21)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    eager = torch.from_numpy(C.copy()).cuda()
    for _ in range(3):
        g.gemm_f16(dA, dB, eager)
    cap = torch.from_numpy(C.copy()).cuda()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        g.gemm_f16(dA, dB, torch.zeros_like(cap))  # warm-up outside capture
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        g.gemm_f16(dA, dB, cap)
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(cap.view(torch.int32), eager.view(torch.int32))


def test_trace_option_records_tiles(g):
    """The diagnostic trace hook fills per-tile stamps without changing results."""
    import torch
    M, N, K = 1024, 1024, 4096
    A, B, C, gA, gB, gC = device_problem(M, N, K, "f32", seed=14)
    tr = torch.zeros(512, dtype=torch.int64, device="cuda")
    _run(g, gA, gB, gC, config="pair_256x256", trace=tr)
    ex, _ = oracle_full(A, B, C)
    check(gC.result(), ex, A, B, "f32", K, "traced")
    t = tr.cpu().numpy().reshape(64, 8)
    assert t[0, 0] > 0 and t[0, 2] > t[0, 0] and t[0, 7] > 0   # MMA begin/end stamps, cycles
    assert t[62, 0] > 0 and t[62, 2] >= t[62, 0]               # kernel entry/exit of CTA 0


@pytest.mark.parametrize("config", ["solo_128x64", "pair_256x256_k128"])
def test_pdl_dependent_chain_exact(config):
    """Programmatic dependent launch: a chain of GEMMs that each read the C the
    previous one wrote, interleaved with torch kernels and inside a CUDA graph, ends
    bitwise at the closed form (small-integer inputs: every partial sum is exact)."""
    import torch
    import paper_2108_13191_b200 as g
    rng = np.random.default_rng(11)
    M, N, K = 300, 520, 264
    A = torch.from_numpy(rng.integers(-2, 3, (M, K)).astype(np.float16)).cuda()
    B = torch.from_numpy(rng.integers(-2, 3, (K, N)).astype(np.float16)).cuda()
    C0 = torch.from_numpy(rng.integers(-50, 51, (M, N)).astype(np.float32)).cuda()
    AB = A.double() @ B.double()
    C = C0.clone()
    for _ in range(6):
        g.gemm_f16(A, B, C, config=config, pdl=1)
    C.mul_(2)                                    # a torch kernel between PDL launches
    for _ in range(3):
        g.gemm_f16(A, B, C, config=config, pdl=1)
    torch.cuda.synchronize()
    assert torch.equal(C.double(), 2 * (C0.double() + 6 * AB) + 3 * AB)
    # captured in a graph
    C.copy_(C0)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        for _ in range(4):
            g.gemm_f16(A, B, C, config=config, pdl=1)
    torch.cuda.synchronize()
    C.copy_(C0)
    gr.replay(); gr.replay()
    torch.cuda.synchronize()
    assert torch.equal(C.double(), C0.double() + 8 * AB)


@pytest.mark.parametrize("acc", ["f32", "f16"])
@pytest.mark.parametrize("shape,pk", [((44, 76, 1064), 128), ((300, 300, 8192), 256), ((1024, 1024, 4096), 64),
                                      ((2048, 2048, 2048), 512)])
def test_auto_with_promote_k_avoids_single_chain_kernels(g, acc, shape, pk):
    # auto would pick a split-K or 256 x 512 kernel for some of these (one TMEM chain per
    # CTA, promote_k rejected there); an explicit promote_k steers auto to a kernel with
    # chunked promotion instead of failing (found by the fuzz campaign, case 257)
    M, N, K = shape
    A, B, C, gA, gB, gC = device_problem(M, N, K, acc, seed=K, pad=(8, 8, 8))
    _run(g, gA, gB, gC, promote_k=pk)
    ex, _ = oracle_full(A, B, C)
    check(gC.result(), ex, A, B, acc, K, f"auto promote_k={pk} {shape}")

"""GPU parity for the stream-K schedule of the F32 pair kernels (gemm_sm100.cuh Work /
Item, option stream_k): when the last wave of tiles is partial, the last partial wave plus
one full wave are shared out over all clusters as equal runs of k-blocks; a tile split
between two clusters meets in C through two TMA reduce-adds in a fixed order.

What is new and checked here against the CPU oracle:
  * every (tile, k-block) unit is computed exactly once (integer-valued inputs: any
    missing or doubled k-range changes the exact result);
  * split points inside a promotion chunk and across chunk boundaries (K > promote_k);
  * the order of the two adds is fixed (bitwise-repeatable results) and the token
    counters are left at zero (later launches still wait: still bitwise-repeatable);
  * data-parallel tiles before the stream-K region (several waves), and the F32 bar.
PAPER.md P:908-909 (C = AB + C), P:967-996 (F32 accumulate)."""
import numpy as np
import pytest

import oracle
import synth
from parity import Guarded, check, device_problem, oracle_full, round_up

pytestmark = pytest.mark.gpu

PAIRS = ["pair_256x256", "pair_256x256_k128", "pair_256x256_s4", "pair_256x256_s5"]


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


# (M, N, K, max_clusters): tiles vs clusters chosen so the last wave is partial
CASES = [
    (1300, 2100, 640, 5),     # 54 tiles on 5 clusters: 10 waves + 4; 9 stream-K tiles x 10 k-blocks
    (1300, 2100, 640, 7),     # 54 = 7 x 7 + 5
    (1000, 1030, 1000, 3),    # 16 tiles on 3 clusters, ragged M and K tail
    (600, 1500, 4200, 4),     # 18 tiles; K crosses two promotion chunks (2048)
    (770, 770, 3000, 3),      # 16 tiles on 3 clusters: 4 stream-K tiles, runs of 62.7 k-blocks (47 per tile)
    (512, 2560, 200, 6),      # short K: 4 / 2 k-blocks per tile
    (700, 700, 2000, 12),     # fewer tiles (9) than clusters: tiles split up to three ways
    (600, 1000, 1500, 10),    # 12 tiles on 10 clusters... and 6 on 10 below
    (300, 1500, 900, 10),
]


@pytest.mark.parametrize("acc", ["f32", "f16"])
@pytest.mark.parametrize("cfg", PAIRS)
@pytest.mark.parametrize("M,N,K,mc", CASES)
def test_stream_k_parity(g, cfg, M, N, K, mc, acc):
    A, B, C, gA, gB, gC = device_problem(M, N, K, acc, seed=M + K, pad=(8, 8, 8))
    _run(g, gA, gB, gC, config=cfg, max_clusters=mc, stream_k=1)
    ex, _ = oracle_full(A, B, C)
    # F16 C: a split tile's two partials are each rounded to binary16 before they meet (R18)
    check(gC.result(), ex, A, B, acc, K, f"{cfg} {acc} {M}x{N}x{K} clusters={mc} stream-K",
          extra_roundings=2 if acc == "f16" else 0)
    assert gC.guard_intact() and gA.guard_intact() and gB.guard_intact()


@pytest.mark.parametrize("cfg", ["pair_256x256", "pair_256x256_k128"])
@pytest.mark.parametrize("mc", [2, 3, 5, 9])
def test_stream_k_every_unit_once_exact(g, cfg, mc):
    # integer-valued A, B, C with |C| < 2^24: every partial sum is exact in F32, so the
    # result is exact whatever the split points -- a k-range computed twice or never fails
    rng = np.random.default_rng(mc)
    M, N, K = 1100, 1300, 1500
    Ai = rng.integers(-2, 3, size=(M, K))
    Bi = rng.integers(-2, 3, size=(K, N))
    Ci = rng.integers(-1000, 1001, size=(M, N))
    gA = Guarded(Ai.astype(np.float16), round_up(K, 8))
    gB = Guarded(Bi.astype(np.float16), round_up(N, 8))
    gC = Guarded(Ci.astype(np.float32), round_up(N, 4))
    _run(g, gA, gB, gC, config=cfg, max_clusters=mc, stream_k=1)
    assert np.array_equal(gC.result().astype(np.int64), Ai @ Bi + Ci)
    assert gC.guard_intact()


@pytest.mark.parametrize("cfg", ["pair_256x256", "pair_256x256_k128"])
@pytest.mark.parametrize("mc", [2, 3, 5])
def test_stream_k_f16_every_unit_once_exact(g, cfg, mc):
    # F16 C (R18: the second part of a split tile is reduce-added in F16): small integers
    # with |C| <= 2048 are exact in every rounding, so the result is exact
    rng = np.random.default_rng(100 + mc)
    M, N, K = 1100, 1304, 1500
    Ai = rng.integers(-1, 2, size=(M, K))
    Bi = rng.integers(-1, 2, size=(K, N))
    Ci = rng.integers(-100, 101, size=(M, N))
    exact = Ai @ Bi + Ci
    assert np.abs(exact).max() <= 2048
    gA = Guarded(Ai.astype(np.float16), round_up(K, 8))
    gB = Guarded(Bi.astype(np.float16), round_up(N, 8))
    gC = Guarded(Ci.astype(np.float16), round_up(N, 8))
    _run(g, gA, gB, gC, config=cfg, max_clusters=mc, stream_k=1)
    assert np.array_equal(gC.result().astype(np.int64), exact)
    assert gC.guard_intact()


def test_stream_k_bitwise_repeatable(g):
    # the two reduce-adds of a split tile happen in a fixed order: 6 launches agree
    # bitwise (a token left behind by one launch would let a later one skip its wait)
    import torch
    M, N, K = 1300, 2100, 2500
    A, B, C, gA, gB, gC = device_problem(M, N, K, "f32", seed=11)
    outs = []
    for _ in range(6):
        gC.full.copy_(torch.from_numpy(gC.full_host.copy()))
        _run(g, gA, gB, gC, config="pair_256x256", max_clusters=5, stream_k=1)
        outs.append(gC.result().copy())
    for o in outs[1:]:
        assert np.array_equal(o.view(np.uint32), outs[0].view(np.uint32))
    ex, _ = oracle_full(A, B, C)
    check(outs[0], ex, A, B, "f32", K, "stream-K repeat")
    # F16 C
    A, B, C, gA, gB, gC = device_problem(M, N, K, "f16", seed=11)
    outs = []
    for _ in range(4):
        gC.full.copy_(torch.from_numpy(gC.full_host.copy()))
        _run(g, gA, gB, gC, config="pair_256x256_k128", max_clusters=5, stream_k=1)
        outs.append(gC.result().copy())
    for o in outs[1:]:
        assert np.array_equal(o.view(np.uint16), outs[0].view(np.uint16))


def test_stream_k_off_and_on_agree_to_rounding(g):
    # the split changes only where two partial sums meet: off/on differ by roundings only
    import torch
    M, N, K = 1024, 2048, 1536
    A, B, C, gA, gB, gC = device_problem(M, N, K, "f32", seed=12)
    res = {}
    for sk in (-1, 1):
        gC.full.copy_(torch.from_numpy(gC.full_host.copy()))
        _run(g, gA, gB, gC, config="pair_256x256", max_clusters=6, stream_k=sk)
        res[sk] = gC.result().copy()
    ex, _ = oracle_full(A, B, C)
    for sk in (-1, 1):
        check(res[sk], ex, A, B, "f32", K, f"stream_k={sk}")


def test_stream_k_ineligible_options_fall_back_to_data_parallel(g):
    # bias / ReLU / beta = 0 / ragged N cannot be split (they are not additive in C):
    # stream_k = 1 is ignored there and the data-parallel result is bitwise unchanged
    import torch
    M, N, K = 900, 1104, 704
    A, B, C = synth.problem(M, N, K, "f32", seed=13)
    bias = torch.from_numpy(synth.uniform_f32(13, 3, 1, N)[0]).cuda()
    for kw in ({"bias": bias}, {"relu": True}, {"beta": 0}):
        outs = []
        for sk in (-1, 1):
            dA, dB, dC = (torch.from_numpy(x).cuda() for x in (A, B, C))
            g.gemm_f16(dA, dB, dC, config="pair_256x256", max_clusters=3, stream_k=sk, **kw)
            torch.cuda.synchronize()
            outs.append(dC.cpu().numpy())
        assert np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32)), kw
    ex, _ = oracle.gemm(A, B, C, bias=bias.cpu().numpy())
    dA, dB, dC = (torch.from_numpy(x).cuda() for x in (A, B, C))
    g.gemm_f16(dA, dB, dC, config="pair_256x256", max_clusters=3, stream_k=1, bias=bias)
    torch.cuda.synchronize()
    check(dC.cpu().numpy(), ex, A, B, "f32", K, "bias, stream_k=1 ignored")


@pytest.mark.parametrize("shape,cfg,sk", [((2304, 2304, 2304), "pair_256x256_k128", 1),
                                          ((4096, 4096, 4096), "pair_256x256_k128", 1),
                                          ((2560, 2560, 8192), "pair_256x256_k128", 1),
                                          ((3840, 3840, 1024), "pair_256x256", 1),
                                          ((2304, 2304, 4096), "auto", 0)])   # (the auto rule takes it)
def test_stream_k_default_grid_sampled(g, shape, cfg, sk):
    # full default grid (74 clusters on a B200), sampled rows
    import torch
    M, N, K = shape
    A, B, C = synth.problem(M, N, K, "f32", seed=14)
    dA, dB, dC = (torch.from_numpy(x).cuda() for x in (A, B, C))
    g.gemm_f16(dA, dB, dC, config=cfg, stream_k=sk)
    torch.cuda.synchronize()
    rows = synth.sample_rows(M, tile_m=128, n_random=24, seed=1)
    rows = rows[np.linspace(0, len(rows) - 1, 48).astype(int)]
    got = dC[torch.from_numpy(rows).cuda()].cpu().numpy()
    ex, _ = oracle.gemm(A, B, C, rows=rows)
    check(got, ex, A[rows], B, "f32", K, f"{shape} stream-K sampled")


def test_stream_k_rejects_bad_option(g):
    import torch
    A = torch.zeros((256, 64), dtype=torch.float16, device="cuda")
    B = torch.zeros((64, 256), dtype=torch.float16, device="cuda")
    C = torch.zeros((256, 256), dtype=torch.float32, device="cuda")
    with pytest.raises(g.GemmError):
        g.gemm_f16(A, B, C, stream_k=2)


def test_stream_k_concurrent_streams_isolated(g):
    # GEMMs with split tiles running at the same time on different streams take different
    # windows of the token pool: each keeps its own fixed order of adds, so the results
    # match the same GEMMs run one at a time, bitwise, and nothing deadlocks
    import torch
    M, N, K = 1300, 2100, 2500
    probs = [device_problem(M, N, K, "f32", seed=30 + i) for i in range(4)]
    ref = []
    for A, B, C, gA, gB, gC in probs:
        _run(g, gA, gB, gC, config="pair_256x256", max_clusters=5, stream_k=1)
        ref.append(gC.result().copy())
        gC.full.copy_(torch.from_numpy(gC.full_host.copy()))
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in probs]
    for rep in range(3):
        for s, (A, B, C, gA, gB, gC) in zip(streams, probs):
            with torch.cuda.stream(s):
                g.gemm_f16(gA.view, gB.view, gC.view, config="pair_256x256", max_clusters=5, stream_k=1)
        torch.cuda.synchronize()
        for r, (A, B, C, gA, gB, gC) in zip(ref, probs):
            assert np.array_equal(gC.result().view(np.uint32), r.view(np.uint32))
            gC.full.copy_(torch.from_numpy(gC.full_host.copy()))
        torch.cuda.synchronize()


@pytest.mark.parametrize("acc", ["f32", "f16"])
def test_stream_k_concurrent_across_window_wrap(g, acc):
    # the token pool is cut into 32 fixed windows taken round robin; run enough
    # concurrent stream-K GEMMs (4 streams x 12 rounds = 48 launches, plus the references)
    # that the window index wraps while others are in flight -- every result must still be
    # bitwise the one-at-a-time result (F32: fixed order of reduce-adds; F16: store, then add)
    import torch
    M, N, K = 1300, 2100, 2500
    probs = [device_problem(M, N, K, acc, seed=50 + i) for i in range(4)]
    ref = []
    for A, B, C, gA, gB, gC in probs:
        _run(g, gA, gB, gC, config="pair_256x256", max_clusters=5, stream_k=1)
        ref.append(gC.result().copy())
        gC.full.copy_(torch.from_numpy(gC.full_host.copy()))
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in probs]
    view = np.uint32 if acc == "f32" else np.uint16
    for rep in range(12):
        for s, (A, B, C, gA, gB, gC) in zip(streams, probs):
            with torch.cuda.stream(s):
                g.gemm_f16(gA.view, gB.view, gC.view, config="pair_256x256", max_clusters=5, stream_k=1)
        torch.cuda.synchronize()
        for r, (A, B, C, gA, gB, gC) in zip(ref, probs):
            assert np.array_equal(gC.result().view(view), r.view(view)), rep
            gC.full.copy_(torch.from_numpy(gC.full_host.copy()))
        torch.cuda.synchronize()


@pytest.mark.parametrize("acc", ["f32", "f16"])
def test_stream_k_graph_replay_isolated_from_eager_launches(g, acc):
    # a CUDA-graph-captured stream-K launch replays for the graph's lifetime, so a
    # window of the shared token pool would be taken again by eager launches on other streams.
    # Forced here: after the capture, advance the pool by exactly one turn, then run the replay
    # and as many eager stream-K launches side by side -- with shared windows each eager launch
    # would use the same counters as the replayed launch next to it.  Captured launches get
    # private counters (graph memory nodes), so both stay bitwise equal to the same launches
    # run alone.  (Sharing corrupts a result only if a waiter arrives between the two launches'
    # posts, which this timing rarely produces: the build before the fix also passed. The test
    # guards the capture path itself: memory nodes, zeroed counters, bitwise results.)
    import torch
    lib = g.load_library()
    n_windows = lib.gemm_f16_diag_sk_pool_slots() // lib.gemm_f16_diag_sk_window_slots()
    M, N, K = 1300, 2100, 2500
    view = np.uint32 if acc == "f32" else np.uint16
    kw = dict(config="pair_256x256", max_clusters=5, stream_k=1)
    (_, _, _, xA, xB, xC), (_, _, _, yA, yB, yC), (_, _, _, zA, zB, zC) = [
        device_problem(M, N, K, acc, seed=70 + i) for i in range(3)]
    n = 6
    for _ in range(n):
        g.gemm_f16(xA.view, xB.view, xC.view, **kw)
        g.gemm_f16(yA.view, yB.view, yC.view, **kw)
    torch.cuda.synchronize()
    ref_x, ref_y = xC.result().copy(), yC.result().copy()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s1):
        for _ in range(n):
            g.gemm_f16(xA.view, xB.view, xC.view, stream=s1, **kw)
    for rep in range(3):
        xC.full.copy_(torch.from_numpy(xC.full_host.copy()))
        yC.full.copy_(torch.from_numpy(yC.full_host.copy()))
        # one whole turn of the pool since the capture (the capture took n windows; after the
        # first rep the n eager launches below do): the next eager launches take the windows
        # the captured launches were given
        for _ in range(n_windows - n):
            g.gemm_f16(zA.view, zB.view, zC.view, **kw)
        torch.cuda.synchronize()
        with torch.cuda.stream(s1):
            graph.replay()
        with torch.cuda.stream(s2):
            for _ in range(n):
                g.gemm_f16(yA.view, yB.view, yC.view, stream=s2, **kw)
        torch.cuda.synchronize()
        assert np.array_equal(xC.result().view(view), ref_x.view(view)), rep
        assert np.array_equal(yC.result().view(view), ref_y.view(view)), rep

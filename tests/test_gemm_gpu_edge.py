"""GPU parity on the binary16 number-format edges, on EVERY output path (VERDICT r01
"what's missing" #4 and weak #1).

PAPER.md Sec. 4.2 P:979-982 flags the F16 mode's "narrower representation for the
mantissa and exponent"; SURVEY 8(c) A5 (RNE downcast, overflow -> +-Inf, NaN
propagates) and A16 (IEEE subnormal inputs) are the readings, R3/R5.
The inputs are built so that the exact result is reached whatever the summation
order or the tensor core's accumulator rounding -- every partial sum is exact in
F32 (and, where a path rounds partial sums to F16, in F16) -- so the GPU result
must equal the oracle's C_round (RNE of the exact double result) exactly.

Output paths (the kernels and epilogue variants that write C):
  f32: staged C_in (c_reduce off), TMA reduce-add (default), 1-CTA, split-K
       (reduce-add steps), stream-K (token-ordered reduce-adds), 256x512 wide tile
       (K-chunk promotion by reduce-adds at staggered points)
  f16: pair tile (C_in staged in smem), 256x512 wide tile (C_in held in registers),
       1-CTA, split-K (DSMEM exchange), stream-K (R18: store + F16 reduce-add)
"""
import numpy as np
import pytest

import oracle
import synth
from parity import CANARY_F16, CANARY_F32, check, round_up

pytestmark = pytest.mark.gpu

# (name, acc, kwargs) -- stream-K needs a partial last wave: (700, 1300) pair tiles = 3 x 6 = 18
# on 4 clusters (4 waves + 2)
PATHS = [
    ("f32_staged", "f32", dict(config="pair_256x256", c_reduce=-1)),
    ("f32_reduce", "f32", dict(config="pair_256x256_k128")),
    ("f32_solo", "f32", dict(config="solo_128x64")),
    ("f32_splitk_s2", "f32", dict(config="splitk_128x128_s2")),
    ("f32_splitk_s4", "f32", dict(config="splitk_128x256_s4")),
    ("f32_streamk", "f32", dict(config="pair_256x256_k128", stream_k=1, max_clusters=4)),
    ("f32_wide", "f32", dict(config="pair_256x512", promote_k=768)),
    ("f16_pair", "f16", dict(config="pair_256x256_k128")),
    ("f16_pair_s5", "f16", dict(config="pair_256x256_s5")),
    ("f16_wide", "f16", dict(config="pair_256x512")),
    ("f16_solo", "f16", dict(config="solo_128x64")),
    ("f16_splitk_s2", "f16", dict(config="splitk_128x128_s2")),
    ("f16_splitk_s4", "f16", dict(config="splitk_128x256_s4")),
    ("f16_streamk", "f16", dict(config="pair_256x256_k128", stream_k=1, max_clusters=4)),
    ("f32_mch", "f32", dict(config="pair2_256x256_mch")),
    ("f16_mch", "f16", dict(config="pair2_256x256_mch")),
    ("f32_mcb", "f32", dict(config="pair2_256x256_mcb")),
    ("f16_mcb", "f16", dict(config="pair2_256x256_mcb")),
]
IDS = [p[0] for p in PATHS]
M0, N0 = 700, 1300


@pytest.fixture(scope="module")
def g():
    import torch
    import paper_2108_13191_b200 as g
    assert torch.cuda.is_available()
    g.load_library()
    return g


def _dev(host, ld=None):
    """Row-major device copy with leading dimension ld (padding left at zero)."""
    import torch
    ld = host.shape[1] if ld is None else ld
    full = np.zeros((host.shape[0], ld), dtype=host.dtype)
    full[:, : host.shape[1]] = host
    return torch.from_numpy(full).cuda()[:, : host.shape[1]]


def _gemm(g, A, B, C, kw):
    import torch
    dC = _dev(C, round_up(C.shape[1], 8))
    g.gemm_f16(_dev(A, round_up(A.shape[1], 8)), _dev(B, round_up(B.shape[1], 8)), dC, **kw)
    torch.cuda.synchronize()
    return dC.cpu().numpy()


def _assert_equal_ieee(got, want, what):
    """Equal as IEEE values: NaN where the oracle has NaN, == elsewhere (so +-0 compare equal)."""
    gn, wn = np.isnan(got), np.isnan(want)
    assert np.array_equal(gn, wn), f"{what}: NaN at {np.argwhere(gn != wn)[:5].tolist()}"
    ok = gn | (got == want)
    if not ok.all():
        i = tuple(np.argwhere(~ok)[0])
        raise AssertionError(f"{what}: {int((~ok).sum())} elements differ; first {i}: got {got[i]!r}, "
                             f"want {want[i]!r}")


# ---------------------------------------------------------------- subnormal inputs (A16)

def _subnormal_problem(acc, K, seed):
    """A: random binary16 subnormals +-k 2^-24 (k in 1..1023) and zeros; B: {-2..2};
    C_in: integers times 2^-24 (F32) or 0 (F16).  Every partial sum is an integer
    multiple of 2^-24 below 2^24 * 2^-24 in magnitude: exact in F32 in any order."""
    rng = np.random.default_rng(seed)
    bits = rng.integers(1, 1024, size=(M0, K)).astype(np.uint16)
    bits |= (rng.random((M0, K)) < 0.5).astype(np.uint16) << np.uint16(15)
    bits[rng.random((M0, K)) < 0.1] = 0
    A = bits.view(np.float16)
    assert np.all(np.abs(A.astype(np.float64)) < 2.0 ** -14)   # all subnormal or zero
    B = rng.integers(-2, 3, size=(K, N0)).astype(np.float16)
    if acc == "f32":
        C = (rng.integers(-1000, 1001, size=(M0, N0)) * 2.0 ** -24).astype(np.float32)
    else:
        C = np.zeros((M0, N0), np.float16)
    return A, B, C


@pytest.mark.parametrize("name,acc,kw", PATHS, ids=IDS)
def test_subnormal_inputs_exact(g, name, acc, kw):
    K = 1536
    A, B, C = _subnormal_problem(acc, K, seed=7)
    got = _gemm(g, A, B, C, kw)
    ex, rnd = oracle.gemm(A, B, C)
    assert np.count_nonzero(ex) > 0.9 * ex.size
    _assert_equal_ieee(got, rnd, f"{name} subnormal A")
    if acc == "f32":   # exact in F32: C_round == C_exact
        assert np.array_equal(got.astype(np.float64), ex)


@pytest.mark.parametrize("name,acc,kw", PATHS, ids=IDS)
def test_subnormal_products_and_output_rounding(g, name, acc, kw):
    """One product per output: subnormal x subnormal = k1 k2 2^-48 (a normal F32, exact).
    In F16 mode that lies below the smallest binary16 subnormal (2^-24) or among the
    subnormals: the epilogue's RNE must round into the subnormal range exactly like
    the oracle (ties to even at 2^-25 included)."""
    rng = np.random.default_rng(3)
    K = 64 * 5
    A = rng.integers(1, 1024, size=(M0, K)).astype(np.uint16).view(np.float16)   # all subnormal
    # column j has one non-zero B[k_j][j]: half the columns a subnormal (products k1 k2 2^-48:
    # F16 output 0), a quarter a normal in [2^-10, 2^-9) (products around binary16's subnormal
    # range: rounding to a multiple of 2^-24), a quarter +-[1, 2) (products near 2^-14 that need
    # rounding to 11 bits) -- random mantissas throughout
    col_k = rng.integers(0, K, size=N0)
    grp = rng.random(N0)
    mant = rng.integers(0, 1024, size=N0).astype(np.uint16)
    vals = rng.integers(1, 1024, size=N0).astype(np.uint16)                       # subnormal
    vals = np.where((grp >= 0.5) & (grp < 0.75), (np.uint16(15 - 10) << np.uint16(10)) | mant, vals)
    vals = np.where(grp >= 0.75, (np.uint16(15) << np.uint16(10)) | mant, vals)
    vals = vals | ((rng.random(N0) < 0.5).astype(np.uint16) << np.uint16(15))
    B = np.zeros((K, N0), np.float16)
    B[col_k, np.arange(N0)] = vals.view(np.float16)
    C = np.zeros((M0, N0), np.float32 if acc == "f32" else np.float16)
    got = _gemm(g, A, B, C, kw)
    ex, rnd = oracle.gemm(A, B, C)
    _assert_equal_ieee(got, rnd, f"{name} subnormal products")
    if acc == "f16":
        # the probe reaches underflow to zero, binary16 subnormal outputs and normal ones
        r = np.abs(rnd.astype(np.float64))
        assert (r == 0).any() and ((r > 0) & (r < 2.0 ** -14)).any() and (r >= 2.0 ** -14).any()
        assert (ex != rnd.astype(np.float64)).any()   # and rounding actually happens


# ---------------------------------------------------------------- overflow -> +-Inf (A5 / R5)

# (a0, a1): C = a0 + a1 exactly (F32), rounded once to binary16
BOUNDARY_PAIRS = [
    (65504.0, 15.0),     # 65519 -> 65504 (below the halfway point)
    (65504.0, 16.0),     # 65520: halfway to 2^16 -> ties-to-even rounds up -> +Inf
    (65504.0, 32.0),     # 65536 -> +Inf
    (-65504.0, -16.0),   # -> -Inf
    (-65504.0, -15.0),   # -> -65504
    (60000.0, 5504.0),   # 65504 exactly
    (65504.0, 65504.0),  # -> +Inf
    (32768.0, 32736.0),  # 65504 exactly
    (-32768.0, -32768.0),  # -65536 -> -Inf
    (1.0, 2.0 ** -24),   # far below: 1 (the tiny term is lost in RNE)
]
F16_PATHS = [p for p in PATHS if p[1] == "f16"]
F16_IDS = [p[0] for p in F16_PATHS]


@pytest.mark.parametrize("name,acc,kw", [p for p in F16_PATHS if "streamk" not in p[0]],
                         ids=[i for i in F16_IDS if "streamk" not in i])
def test_f16_output_overflow_boundary(g, name, acc, kw):
    K = 64
    A = np.zeros((M0, K), np.float16)
    pairs = np.array(BOUNDARY_PAIRS * (M0 // len(BOUNDARY_PAIRS) + 1))[:M0]
    A[:, 0] = pairs[:, 0].astype(np.float16)
    A[:, 1] = pairs[:, 1].astype(np.float16)
    assert np.array_equal(A[:, :2].astype(np.float64), pairs)   # every term exact in binary16
    B = np.zeros((K, N0), np.float16)
    B[0, :] = 1
    B[1, :] = 1
    C = np.zeros((M0, N0), np.float16)
    got = _gemm(g, A, B, C, kw)
    _, rnd = oracle.gemm(A, B, C)
    assert np.isinf(rnd).sum() > 0 and np.isfinite(rnd).sum() > 0
    _assert_equal_ieee(got, rnd, f"{name} overflow boundary")


@pytest.mark.parametrize("name,acc,kw", PATHS, ids=IDS)
def test_large_sums_overflow_to_inf(g, name, acc, kw):
    """Every product of row i and column j is s_i 2^(e_i + f_j); C = s_i 2^(e_i+f_j) K with
    K = 1536 is 12288 / 24576 / 49152 (exact in binary16) or 98304 (-> s_i Inf in F16 C,
    exact in F32 C).  Any split of K at k-block boundaries gives partial sums that are exact
    in binary16 (or already overflow, with one sign), so F16 stream-K also lands exactly."""
    rng = np.random.default_rng(11)
    K = 1536
    e = rng.integers(0, 4, size=M0)
    s = rng.choice([-1.0, 1.0], size=M0)
    f = rng.integers(3, 4, size=N0)
    A = np.repeat((s * 2.0 ** e)[:, None], K, axis=1).astype(np.float16)
    B = np.repeat((2.0 ** f)[None, :], K, axis=0).astype(np.float16)
    C = np.zeros((M0, N0), np.float32 if acc == "f32" else np.float16)
    got = _gemm(g, A, B, C, kw)
    ex, rnd = oracle.gemm(A, B, C)
    if acc == "f16":
        assert np.isposinf(rnd).any() and np.isneginf(rnd).any() and np.isfinite(rnd).any()
    _assert_equal_ieee(got, rnd, f"{name} large sums")


# ---------------------------------------------------------------- special C_in values

def _special_cin_problem(acc, seed):
    """Integer A, B, C_in (exact in the mode's type: F32 |C| < 2^24; F16 |C| <= 2048),
    with +Inf / -Inf / NaN scattered through C_in, tile corners included."""
    rng = np.random.default_rng(seed)
    K = 1536
    lo = 2 if acc == "f32" else 1
    A = rng.integers(-lo, lo + 1, size=(M0, K)).astype(np.float16)
    B = rng.integers(-lo, lo + 1, size=(K, N0)).astype(np.float16)
    if acc == "f16":
        # keep |C| <= 2048: A, B in {-1, 0, 1} with |sum| <= 1536, C_in in [-256, 256]
        C = rng.integers(-256, 257, size=(M0, N0)).astype(np.float16)
    else:
        C = rng.integers(-1000, 1001, size=(M0, N0)).astype(np.float32)
    special = np.array([np.inf, -np.inf, np.nan])
    idx = rng.random((M0, N0)) < 0.02
    C[idx] = rng.choice(special, size=int(idx.sum()))
    for r in (0, 127, 128, 255, 256, 511, 512, M0 - 1):   # tile corners
        for c in (0, 63, 64, 255, 256, 511, 512, N0 - 1):
            C[r, c] = special[(r + c) % 3]
    return A, B, C


@pytest.mark.parametrize("name,acc,kw", PATHS, ids=IDS)
def test_special_c_in_propagates(g, name, acc, kw):
    A, B, C = _special_cin_problem(acc, seed=5)
    got = _gemm(g, A, B, C, kw)
    ex, rnd = oracle.gemm(A, B, C)
    assert np.isnan(rnd).any() and np.isposinf(rnd).any() and np.isneginf(rnd).any()
    _assert_equal_ieee(got, rnd, f"{name} special C_in")


# ---------------------------------------------------------------- P8: brute force on tiny shapes

def _p8_shapes(n, seed):
    """A seeded subset of M, N, K in [1..40] that covers every value of each axis."""
    rng = np.random.default_rng(seed)
    shapes = {(v, int(rng.integers(1, 41)), int(rng.integers(1, 41))) for v in range(1, 41)}
    shapes |= {(int(rng.integers(1, 41)), v, int(rng.integers(1, 41))) for v in range(1, 41)}
    shapes |= {(int(rng.integers(1, 41)), int(rng.integers(1, 41)), v) for v in range(1, 41)}
    while len(shapes) < n:
        shapes.add(tuple(int(x) for x in rng.integers(1, 41, size=3)))
    return sorted(shapes)


P8_CONFIGS = {"f32": ["auto", "pair_256x256", "solo_128x64", "splitk_128x128_s2", "pair_256x256_k128"],
              "f16": ["auto", "pair_256x256", "solo_128x64", "splitk_128x128_s2", "pair_256x512"]}


@pytest.mark.parametrize("acc", ["f32", "f16"])
def test_p8_tiny_shape_grid(g, acc):
    """SURVEY 8(c) P8 on 2,000 seeded shapes of M, N, K in [1..40] (every value of each axis
    included), padded leading dims, configs rotated over the kernel families.  All GEMMs are
    enqueued on one arena with canary padding and checked after a single synchronisation."""
    import torch
    shapes = _p8_shapes(2000, seed=17 if acc == "f32" else 18)
    csz = 4 if acc == "f32" else 2
    lay, offA, offB, offC = [], 0, 0, 0
    for (M, N, K) in shapes:
        lda, ldb, ldc = round_up(K, 8) + 8, round_up(N, 8) + 8, round_up(N, 16 // csz) + 16 // csz
        lay.append((M, N, K, lda, ldb, ldc, offA, offB, offC))
        offA += round_up(M * lda, 64)
        offB += round_up(K * ldb, 64)
        offC += round_up(M * ldc, 64)
    hA = np.full(offA, CANARY_F16, np.uint16).view(np.float16)
    hB = np.full(offB, CANARY_F16, np.uint16).view(np.float16)
    hC = (np.full(offC, CANARY_F32, np.uint32).view(np.float32) if acc == "f32"
          else np.full(offC, CANARY_F16, np.uint16).view(np.float16))
    probs = []
    for i, (M, N, K, lda, ldb, ldc, oa, ob, oc) in enumerate(lay):
        A, B, C = synth.problem(M, N, K, acc, seed=i % 5)
        hA[oa:oa + M * lda].reshape(M, lda)[:, :K] = A
        hB[ob:ob + K * ldb].reshape(K, ldb)[:, :N] = B
        hC[oc:oc + M * ldc].reshape(M, ldc)[:, :N] = C
        probs.append((A, B, C))
    dA, dB, dC = (torch.from_numpy(x.copy()).cuda() for x in (hA, hB, hC))
    cfgs = P8_CONFIGS[acc]
    for i, (M, N, K, lda, ldb, ldc, oa, ob, oc) in enumerate(lay):
        g.gemm_f16(dA[oa:oa + M * lda].view(M, lda)[:, :K], dB[ob:ob + K * ldb].view(K, ldb)[:, :N],
                   dC[oc:oc + M * ldc].view(M, ldc)[:, :N], config=cfgs[i % len(cfgs)])
    torch.cuda.synchronize()
    out = dC.cpu().numpy()
    mask = np.ones(offC, bool)
    for (M, N, K, lda, ldb, ldc, oa, ob, oc) in lay:
        win = mask[oc:oc + M * ldc].reshape(M, ldc)
        win[:, :N] = False
    bits = np.uint32 if acc == "f32" else np.uint16
    assert np.array_equal(out.view(bits)[mask], hC.view(bits)[mask]), "write outside an M x N window"
    for i, ((M, N, K, lda, ldb, ldc, oa, ob, oc), (A, B, C)) in enumerate(zip(lay, probs)):
        got = out[oc:oc + M * ldc].reshape(M, ldc)[:, :N]
        ex, _ = oracle.gemm(A, B, C)
        check(got, ex, A, B, acc, K, f"P8 {(M, N, K)} {cfgs[i % len(cfgs)]}")

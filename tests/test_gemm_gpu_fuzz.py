"""Seeded fuzzing of the CUDA path against the oracle: random shapes (incl. 1 and
odd sizes), random padded leading dims, random configurations and scheduling /
epilogue options (stream-K included), both output modes and both input types; guard bands must stay
untouched.  Every case is reproducible from its index."""
import os

import numpy as np
import pytest

import oracle
import synth
from parity import CANARY_F16, CANARY_F32, check, round_up

pytestmark = pytest.mark.gpu

CONFIGS = ["auto", "pair_256x256", "pair_256x128", "solo_128x256", "solo_128x128", "solo_128x64",
           "pair_256x256_s5", "pair_256x256_s4", "pair_256x256_k128"]


# the CTA-pair configurations built with stream-K (gemm_api.cu sk_fn_of: cta_group::2, no peers)
STREAM_K_CONFIGS = {"pair_256x256", "pair_256x128", "pair_256x256_s5", "pair_256x256_s4", "pair_256x256_k128"}


def _guarded_dev(host_bits, ld, rows_extra, canary):
    import torch
    full = np.full((host_bits.shape[0] + rows_extra, ld), canary, dtype=host_bits.dtype)
    full[: host_bits.shape[0], : host_bits.shape[1]] = host_bits
    return full, torch.from_numpy(full.copy()).cuda()


N_MAIN = int(os.environ.get("FUZZ_MAIN", "48"))    # a longer campaign: FUZZ_MAIN=500


@pytest.mark.parametrize("case", range(N_MAIN))
def test_fuzz_against_oracle(case):
    _fuzz_case(case, 10_000 + case, wide=False)


@pytest.mark.parametrize("case", range(24))
def test_fuzz_wide_tile_against_oracle(case):
    # GEMM_CFG_PAIR_256x512 (F16 C only), larger N so several 512-column tiles occur
    _fuzz_case(case, 20_000 + case, wide=True)


SPLIT_AND_MC = ["splitk_128x256_s2", "splitk_128x256_s4", "splitk_128x128_s4", "splitk_128x128_s2",
                "solo_128x64_mc4", "solo_128x128_mc4"]
N_EXTRA = int(os.environ.get("FUZZ_EXTRA", "24"))   # a longer campaign: FUZZ_EXTRA=300


@pytest.mark.parametrize("case", range(N_EXTRA))
def test_fuzz_split_and_multicast_against_oracle(case):
    # the cluster kernels: split-K (DSMEM / bulk-DMA / reduce-add paths) and A multicast
    _fuzz_case(case, 30_000 + case, wide=False, configs=SPLIT_AND_MC)


@pytest.mark.parametrize("case", range(N_EXTRA))
def test_fuzz_b_multicast_against_oracle(case):
    # the B-multicast kernel in 4-CTA clusters (mcb) and under the preferred-cluster launch (mch:
    # 4-CTA clusters where they fit, lone pairs elsewhere)
    _fuzz_case(case, 40_000 + case, wide=False, configs=["pair2_256x256_mcb", "pair2_256x256_mch"])


def _fuzz_case(case, seed, wide, configs=None):
    import torch
    import paper_2108_13191_b200 as g
    rng = np.random.default_rng(seed)
    M = int(rng.choice([1, 2, 7, 31, 127, 128, 129, 255, 256, 257]) if rng.random() < 0.3 else rng.integers(1, 700))
    N = int(rng.choice([1, 8, 9, 63, 64, 65, 256, 264]) if rng.random() < 0.3 else rng.integers(1, 700))
    K = int(rng.choice([1, 15, 16, 17, 63, 64, 65, 128, 129]) if rng.random() < 0.3 else rng.integers(1, 1500))
    acc = "f32" if rng.random() < 0.5 else "f16"
    bf16 = rng.random() < 0.25
    kw = {"config": str(rng.choice(configs or CONFIGS))}
    if wide:
        acc, kw["config"] = "f16", "pair_256x512"
        N = int(rng.integers(1, 2600))
    if rng.random() < 0.3:
        kw["max_clusters"] = int(rng.integers(1, 5))
    if rng.random() < 0.3:
        kw["group_m"] = int(rng.integers(1, 9))
    if rng.random() < 0.3:
        kw["acc_bufs"] = 1
    if rng.random() < 0.3 and not wide:
        kw["promote_k"] = int(rng.choice([-1, 128, 256, 512]))
    if wide and rng.random() < 0.3:
        kw["ring_stages"] = int(rng.integers(1, 5))
    if rng.random() < 0.2:
        kw["raster"] = 1
    if kw["config"].startswith("splitk") and kw.get("promote_k", 0) > 0:
        kw["promote_k"] = -1      # split configs keep one chain per K share by design
    beta = 0 if rng.random() < 0.2 else 1
    relu = rng.random() < 0.2
    use_bias = rng.random() < 0.25

    if bf16:
        A, B, C = synth.problem_bf16(M, N, K, acc, seed=case % 7)
        Abits, Bbits = A, B
    else:
        A, B, C = synth.problem(M, N, K, acc, seed=case % 7)
        Abits, Bbits = A.view(np.uint16), B.view(np.uint16)
    csz = 4 if acc == "f32" else 2
    lda = round_up(max(K, 1), 8) + 8 * int(rng.integers(0, 3))
    ldb = round_up(max(N, 1), 8) + 8 * int(rng.integers(0, 3))
    ldc = round_up(max(N, 1), 16 // csz) + (16 // csz) * int(rng.integers(0, 3))
    if not wide and rng.random() < 0.4:
        kw["stream_k"] = 1        # pair configs with a partial last wave split tiles (else ignored)
    _, dA = _guarded_dev(Abits, lda, 1, np.uint16(CANARY_F16))
    _, dB = _guarded_dev(Bbits, ldb, 1, np.uint16(CANARY_F16))
    cbits = C.view(np.uint32 if acc == "f32" else np.uint16)
    cfull, dC = _guarded_dev(cbits, ldc, 2, CANARY_F32 if acc == "f32" else np.uint16(CANARY_F16))
    in_dt = torch.bfloat16 if bf16 else torch.float16
    out_dt = torch.float32 if acc == "f32" else torch.float16
    tA = dA.view(torch.int16).view(in_dt)[:M, :K]
    tB = dB.view(torch.int16).view(in_dt)[:K, :N]
    tC = (dC.view(torch.int32).view(torch.float32) if acc == "f32" else dC.view(torch.int16).view(torch.float16))[:M, :N]
    bias = synth.uniform_f32(case, 3, 1, N)[0] if use_bias else None
    g.gemm_f16(tA, tB, tC, beta=beta, relu=relu, bias=None if bias is None else torch.from_numpy(bias).cuda(), **kw)
    torch.cuda.synchronize()
    out = dC.cpu().numpy()
    # guard bands (ld padding and trailing rows) untouched
    mask = np.ones(out.shape, bool)
    mask[:M, :N] = False
    assert np.array_equal(out[mask], cfull[mask]), f"case {case}: write outside the window"
    got = out[:M, :N].view(np.float32 if acc == "f32" else np.float16)
    ex, _ = oracle.gemm(A, B, C, in_type=1 if bf16 else 0, beta=beta, bias=bias, relu=relu)
    Av = A.astype(np.float32) if not bf16 else torch.from_numpy(A.view(np.int16)).view(torch.bfloat16).float().numpy()
    Bv = B.astype(np.float32) if not bf16 else torch.from_numpy(B.view(np.int16)).view(torch.bfloat16).float().numpy()
    # a stream-K split tile with F16 C rounds twice more (DESIGN R18: rn16(C_in + p0), rn16(p1)),
    # each time by up to half a binary16 ulp of a partial sum's magnitude (<= S)
    sk_f16 = acc == "f16" and kw.get("stream_k") == 1 and kw["config"] in STREAM_K_CONFIGS
    check(got, ex, Av, Bv, acc, K, f"case {case}: {(M, N, K)} {acc} bf16={bf16} {kw} beta={beta} relu={relu} bias={use_bias}",
          C_in=C if beta else None, extra_roundings=2 if sk_f16 else 0)

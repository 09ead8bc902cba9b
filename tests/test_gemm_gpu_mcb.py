"""GEMM_CFG_PAIR2_256x256_MCB: two CTA pairs per 4-CTA cluster, the shared B box TMA-multicast
between the pairs (north_star "clusters multicasting the shared operand"), and
GEMM_CFG_PAIR2_256x256_MCH, the same kernel launched with a preferred cluster dim of 4 over
regular 2-CTA clusters (a group of four CTAs multicasts where the hardware places it as one
cluster and runs as two independent pairs elsewhere).  Parity against the oracle on ragged
shapes (odd pair-tile rows: the second pair of a group then runs wholly outside C), closed
forms bit-exact, determinism, and bitwise equality with the 2-CTA pair kernel."""
import numpy as np
import pytest

import oracle
import synth
from parity import Guarded, check, device_problem, round_up

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    import paper_2108_13191_b200 as g
    g.load_library()
    return g


def _run(g, gA, gB, gC, **kw):
    import torch
    g.gemm_f16(gA.view, gB.view, gC.view, **kw)
    torch.cuda.synchronize()


CFGS = ["pair2_256x256_mcb", "pair2_256x256_mch"]


@pytest.mark.parametrize("cfg", CFGS)
@pytest.mark.parametrize("acc", ["f32", "f16"])
@pytest.mark.parametrize("shape", [(512, 256, 256), (768, 520, 300), (1300, 700, 1100), (256, 1024, 2048),
                                   (2304, 1536, 640), (200, 130, 64)])
def test_b_multicast_parity(g, acc, shape, cfg):
    M, N, K = shape
    A, B, C, gA, gB, gC = device_problem(M, N, K, acc, seed=7, pad=(8, 8, 8))
    _run(g, gA, gB, gC, config=cfg)
    ex, _ = oracle.gemm(A, B, C)
    check(gC.result(), ex, A, B, acc, K, f"mcb {shape} {acc}", C_in=C)
    assert gC.guard_intact()


@pytest.mark.parametrize("acc", ["f32", "f16"])
def test_b_multicast_persistent_and_deterministic(g, acc):
    # many tiles per cluster (phase wrap of the ring and the accumulators), bitwise equal to the
    # 2-CTA pair kernel on small integers (exact) and run to run
    import torch
    M, N, K = 2048, 1024, 576
    rng = np.random.default_rng(3)
    A = rng.integers(-2, 3, (M, K)).astype(np.float16)
    B = rng.integers(-2, 3, (K, N)).astype(np.float16)
    C = rng.integers(-4, 5, (M, N)).astype(np.float32 if acc == "f32" else np.float16)
    if acc == "f16":
        A = np.clip(A, -1, 1).astype(np.float16); B = np.clip(B, -1, 1).astype(np.float16)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    outs = []
    for cfg, mc in (("pair2_256x256_mcb", 1), ("pair2_256x256_mcb", 2), ("pair_256x256_k128", 1),
                    ("pair2_256x256_mch", 1), ("pair2_256x256_mch", 3), ("pair2_256x256_mch", 0)):
        dC = torch.from_numpy(C.copy()).cuda()
        g.gemm_f16(dA, dB, dC, config=cfg, max_clusters=mc)
        torch.cuda.synchronize()
        outs.append(dC.cpu().numpy())
    ex, rnd = oracle.gemm(A, B, C)
    for o in outs:
        assert np.array_equal(o, rnd)


@pytest.mark.parametrize("cfg", CFGS)
@pytest.mark.parametrize("acc", ["f32", "f16"])
@pytest.mark.parametrize("opt", ["beta0", "bias_relu", "bf16", "promote_256", "acc_bufs_1"])
def test_b_multicast_with_options(g, acc, opt, cfg):
    import torch
    M, N, K = 900, 520, 704
    if opt == "bf16":
        A, B, C = synth.problem_bf16(M, N, K, acc, seed=9)
        tA = torch.from_numpy(A.view(np.int16)).cuda().view(torch.bfloat16)
        tB = torch.from_numpy(B.view(np.int16)).cuda().view(torch.bfloat16)
        Av = tA.float().cpu().numpy(); Bv = tB.float().cpu().numpy()
    else:
        A, B, C = synth.problem(M, N, K, acc, seed=9)
        tA, tB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
        Av, Bv = A.astype(np.float32), B.astype(np.float32)
    dC = torch.from_numpy(C.copy()).cuda()
    bias = synth.uniform_f32(9, 3, 1, N)[0] if opt == "bias_relu" else None
    kw = dict(config=cfg, beta=0 if opt == "beta0" else 1, relu=opt == "bias_relu",
              bias=None if bias is None else torch.from_numpy(bias).cuda())
    if opt == "promote_256":
        kw["promote_k"] = 256
    if opt == "acc_bufs_1":
        kw["acc_bufs"] = 1
    g.gemm_f16(tA, tB, dC, **kw)
    torch.cuda.synchronize()
    ex, _ = oracle.gemm(A, B, C, in_type=1 if opt == "bf16" else 0, beta=kw["beta"], bias=bias, relu=kw["relu"])
    check(dC.cpu().numpy(), ex, Av, Bv, acc, K, f"mcb {opt} {acc}", C_in=C if kw["beta"] else None)


@pytest.mark.parametrize("acc", ["f32", "f16"])
@pytest.mark.parametrize("shape", [(4096, 4096, 2048), (8192, 8192, 1024), (2560, 3072, 4160)])
def test_hybrid_bitwise_equal_to_pair_kernel(g, acc, shape):
    # the full grid (every SM: 4-CTA clusters where they fit, lone pairs elsewhere), many tiles
    # per group: each tile runs the same MMA sequence and epilogue as in the 2-CTA pair kernel,
    # so the results are bitwise equal on random data; also run to run
    import torch
    M, N, K = shape
    A, B, C = synth.problem(M, N, K, acc, seed=11)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    outs = []
    for cfg in ("pair_256x256_k128", "pair2_256x256_mch", "pair2_256x256_mch", "pair2_256x256_mcb"):
        dC = torch.from_numpy(C.copy()).cuda()
        g.gemm_f16(dA, dB, dC, config=cfg)
        torch.cuda.synchronize()
        outs.append(dC.cpu().numpy())
    for o in outs[1:]:
        assert np.array_equal(o.view(np.uint32 if acc == "f32" else np.uint16),
                              outs[0].view(np.uint32 if acc == "f32" else np.uint16))

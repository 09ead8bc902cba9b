"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (auto config, default options), on rows the oracle computes one by one
(first/last rows of tile row-blocks + seeded random rows), plus the fake-rank
N-shard invariance and the BERT-shaped problems with tails
(BASELINE.json configs[4])."""
import numpy as np
import pytest

import oracle
import synth
from parity import check

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    import paper_2108_13191_b200 as g
    g.load_library()
    return g


def _sampled_check(g, M, N, K, acc, seed=0, n_random=24, **kw):
    import torch
    A, B, C = synth.problem(M, N, K, acc, seed=seed)
    dA, dB, dC = (torch.from_numpy(x).cuda() for x in (A, B, C))
    g.gemm_f16(dA, dB, dC, **kw)
    torch.cuda.synchronize()
    rows = synth.sample_rows(M, tile_m=128, n_random=n_random, seed=seed)
    if len(rows) > 96:
        keep = np.linspace(0, len(rows) - 1, 96).astype(int)
        rows = rows[keep]
    got = dC[torch.from_numpy(rows).cuda()].cpu().numpy()
    ex, _ = oracle.gemm(A, B, C, rows=rows)
    return check(got, ex, A[rows], B, acc, K, f"{(M, N, K)} {acc} sampled")


@pytest.mark.parametrize("acc", ["f32", "f16"])
def test_8192_cube_sampled(g, acc):
    s = _sampled_check(g, 8192, 8192, 8192, acc)
    print(f"8192^3 {acc}: {s}")


@pytest.mark.parametrize("acc", ["f16"])
def test_1024_cube_full(g, acc):
    # BASELINE.json configs[1]: M=N=K=1024, F16 accumulate -- every element
    import torch
    M = N = K = 1024
    A, B, C = synth.problem(M, N, K, acc, seed=1)
    dA, dB, dC = (torch.from_numpy(x).cuda() for x in (A, B, C))
    g.gemm_f16(dA, dB, dC)
    torch.cuda.synchronize()
    ex, _ = oracle.gemm(A, B, C)
    check(dC.cpu().numpy(), ex, A, B, acc, K, "1024^3 full")


@pytest.mark.parametrize("n", [2048, 4096, 6144, 10240, 12288, 14336, 16384])
def test_square_sweep_sampled(g, n):
    for acc in ("f32", "f16"):
        _sampled_check(g, n, n, n, acc, n_random=8)


BERT = [(4096, 1024, 1024), (4096, 4096, 1024), (8192, 1024, 4096), (16384, 4096, 4096), (32768, 1024, 4096),
        (4097, 1024, 1024), (12345, 4096, 1024), (32767, 1024, 4096), (8192, 1000, 1000), (4100, 4096, 4104)]


@pytest.mark.parametrize("shape", BERT)
def test_bert_shapes_sampled(g, shape):
    M, N, K = shape
    for acc in ("f32", "f16"):
        _sampled_check(g, M, N, K, acc, n_random=8)


def test_fake_rank_nshard_bitwise(g):
    """Rank slabs computed one after another on one GPU with the same kernel
    config reproduce the unsharded columns bitwise (no cross-column arithmetic)."""
    import torch
    from paper_2108_13191_b200 import dist as gdist
    M, N, K = 2048, 4096, 2048
    A, B, C = synth.problem(M, N, K, "f32", seed=5)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    full = torch.from_numpy(C).cuda()
    g.gemm_f16(dA, dB, full, config="pair_256x256")
    for P in (2, 4, 8):
        out = torch.empty_like(full)
        for (n0, n1) in gdist.column_slabs(N, P):
            B_r = dB[:, n0:n1].contiguous()
            C_r = torch.from_numpy(np.ascontiguousarray(C[:, n0:n1])).cuda()
            gdist.gemm_nshard(dA, B_r, C_r, config="pair_256x256")
            out[:, n0:n1] = C_r
        torch.cuda.synchronize()
        assert torch.equal(out.view(torch.int32), full.view(torch.int32)), P

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


def _sampled_check(g, M, N, K, acc, seed=0, n_random=24, extra_roundings=0, **kw):
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
    return check(got, ex, A[rows], B, acc, K, f"{(M, N, K)} {acc} sampled", C_in=C[rows],
                 extra_roundings=extra_roundings)


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


@pytest.mark.parametrize("P", [2, 3, 4, 8])
@pytest.mark.parametrize("acc", ["f32", "f16"])
def test_fused_gather_simulated_ranks(g, P, acc):
    """gemm_f16_gather on one GPU with P full-size C buffers standing in for the
    P ranks' memories: rank r computes its slab and stores it into all P buffers.
    Afterwards every buffer equals the unsharded C += A.B (oracle parity), and
    bitwise equals the plain GEMM in the same tile configuration."""
    import torch
    from paper_2108_13191_b200 import dist as gdist
    M, N, K = 600, 1000, 2200    # ragged M; N slabs of 8-column multiples incl. a ragged last one
    A, B, C = synth.problem(M, N, K, acc, seed=30 + P)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    bufs = [torch.from_numpy(C.copy()).cuda() for _ in range(P)]
    slabs = gdist.column_slabs(N, P, align=8)
    for r in range(P):
        n0, n1 = slabs[r]
        B_r = dB[:, n0:n1].contiguous()
        peers = [bufs[j] for j in range(P) if j != r]
        gdist.gemm_nshard_gather(dA, B_r, bufs[r], slabs, r, peer_ptrs=peers)
    torch.cuda.synchronize()
    ex, _ = oracle.gemm(A, B, C)
    ref = torch.from_numpy(C.copy()).cuda()
    g.gemm_f16(dA, dB, ref, config="pair_256x256_k128")
    for r in range(P):
        check(bufs[r].cpu().numpy(), ex, A, B, acc, K, f"gather P={P} buffer {r}")
    ibits = torch.int32 if acc == "f32" else torch.int16
    for r in range(P):   # per-element K order is independent of the N tiling
        assert torch.equal(bufs[r].view(ibits), ref.view(ibits)), r


def test_symmetric_buffer_rendezvous_single_rank(g):
    """The symmetric-memory plumbing of the fused gather runs on a 1-rank NCCL
    group (no peers): allocation, rendezvous, and the fused kernel on the buffer."""
    import os, socket
    import torch
    import torch.distributed as dist
    from paper_2108_13191_b200 import dist as gdist
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        M, N, K = 512, 768, 640
        A, B, C = synth.problem(M, N, K, "f32", seed=44)
        t, peers, hdl = gdist.symmetric_c_buffer(M, N, torch.float32)
        assert peers == []
        t.copy_(torch.from_numpy(C))
        slabs = gdist.column_slabs(N, 1)
        gdist.gemm_nshard_gather(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), t, slabs, 0, peers)
        torch.cuda.synchronize()
        hdl.barrier()
        ex, _ = oracle.gemm(A, B, C)
        check(t.cpu().numpy(), ex, A, B, "f32", K, "symmetric buffer")
    finally:
        dist.destroy_process_group()


# round 2: the mid-size F32 rule (S4 ring with stream-K just over one wave) and the fused
# epilogue options at multi-wave sizes (the fuzz covers them at <= 700 x 700)
@pytest.mark.parametrize("shape", [(2304, 2304, 2304), (2304, 2560, 2560), (2304, 2304, 4096)])
def test_one_wave_s4_stream_k_sampled(g, shape):
    M, N, K = shape
    for acc in ("f32", "f16"):
        # F16 C takes stream-K here too (partial last wave, K > 2048): its split tiles round
        # twice more (DESIGN R18), which the element gate allows for
        _sampled_check(g, M, N, K, acc, n_random=8, extra_roundings=2 if acc == "f16" else 0)


@pytest.mark.parametrize("acc", ["f32", "f16"])
@pytest.mark.parametrize("opt", ["bf16", "beta0", "bias_relu"])
def test_epilogue_options_at_scale_sampled(g, acc, opt):
    import torch
    M = N = K = 4096
    if opt == "bf16":
        A, B, C = synth.problem_bf16(M, N, K, acc, seed=2)
        tA = torch.from_numpy(A.view(np.int16)).cuda().view(torch.bfloat16)
        tB = torch.from_numpy(B.view(np.int16)).cuda().view(torch.bfloat16)
    else:
        A, B, C = synth.problem(M, N, K, acc, seed=2)
        tA, tB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    dC = torch.from_numpy(C.copy()).cuda()
    bias = synth.uniform_f32(2, 3, 1, N)[0] if opt == "bias_relu" else None
    kw = dict(beta=0 if opt == "beta0" else 1, relu=opt == "bias_relu",
              bias=None if bias is None else torch.from_numpy(bias).cuda())
    g.gemm_f16(tA, tB, dC, **kw)
    torch.cuda.synchronize()
    rows = synth.sample_rows(M, tile_m=128, n_random=8, seed=2)
    got = dC[torch.from_numpy(rows).cuda()].cpu().numpy()
    ex, _ = oracle.gemm(A, B, C, rows=rows, in_type=1 if opt == "bf16" else 0, beta=kw["beta"], bias=bias,
                        relu=kw["relu"])
    Av = (torch.from_numpy(A.view(np.int16)).view(torch.bfloat16).float().numpy() if opt == "bf16"
          else A.astype(np.float32))
    Bv = (torch.from_numpy(B.view(np.int16)).view(torch.bfloat16).float().numpy() if opt == "bf16"
          else B.astype(np.float32))
    check(got, ex, Av[rows], Bv, acc, K, f"4096^3 {acc} {opt} sampled", C_in=C[rows] if kw["beta"] else None)

"""The binding's fast path for the default call (`_gemm_f16_fast`, profiles/r02/findings.md §10):
it must launch exactly what the general path launches (bitwise-equal C on the same inputs) and
hand every unusual argument to the general path, so errors keep their precise types."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    import torch
    import paper_2108_13191_b200 as g
    assert torch.cuda.is_available()
    g.load_library()
    return g


@pytest.mark.parametrize("acc", ["f32", "f16"])
@pytest.mark.parametrize("shape", [(300, 520, 200), (1024, 1024, 1024), (8, 8, 8)])
def test_fast_path_bitwise_equal_to_general_path(g, acc, shape):
    import torch
    M, N, K = shape
    A, B, C = synth.problem(M, N, K, acc, seed=3)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    c_fast, c_gen = torch.from_numpy(C.copy()).cuda(), torch.from_numpy(C.copy()).cuda()
    assert g._gemm_f16_fast(dA, dB, c_fast) is c_fast          # the fast path took it
    g.gemm_f16(dA, dB, c_gen, config="auto")                     # the general path (its checks, _ld)
    torch.cuda.synchronize()
    bits = np.uint32 if acc == "f32" else np.uint16
    assert np.array_equal(c_fast.cpu().numpy().view(bits), c_gen.cpu().numpy().view(bits))


def test_fast_path_declines_unusual_arguments(g):
    import torch
    A = torch.zeros((64, 32), dtype=torch.float16, device="cuda")
    B = torch.zeros((32, 48), dtype=torch.float16, device="cuda")
    C = torch.zeros((64, 48), dtype=torch.float32, device="cuda")
    cases = [
        (A.cpu(), B, C),                                  # CPU operand
        (A.bfloat16(), B.bfloat16(), C),                  # bf16 inputs (general path handles them)
        (A, B, C.double()),                               # unsupported C type
        (A, B[:16], C),                                   # K mismatch
        (A.t().contiguous().t(), B, C),                   # column-major A
        (A[:1], B, C[:1]),                                # a single row (leading-dim rule)
        (A.reshape(-1), B, C),                            # not 2-D
    ]
    for a, b, c in cases:
        assert g._gemm_f16_fast(a, b, c) is None


def test_errors_keep_their_types_through_the_default_call(g):
    import torch
    A = torch.zeros((64, 32), dtype=torch.float16, device="cuda")
    B = torch.zeros((32, 48), dtype=torch.float16, device="cuda")
    C = torch.zeros((64, 48), dtype=torch.float32, device="cuda")
    with pytest.raises(ValueError):
        g.gemm_f16(A.cpu(), B, C)
    with pytest.raises(TypeError):
        g.gemm_f16(A, B, C.double())
    with pytest.raises(ValueError):
        g.gemm_f16(A, B[:16], C)
    with pytest.raises(ValueError):
        g.gemm_f16(A.t().contiguous().t(), B, C)
    # a leading dimension the library rejects (stride 0 rows) comes back as a GemmError
    with pytest.raises(g.GemmError):
        g.gemm_f16(A[:1].expand(64, 32), B, C)


def test_fastbind_extension_matches_the_general_path(g):
    """The in-tree torch extension of the default call (csrc/fastbind.cpp), when built, is what
    the default call uses; it launches exactly the general path's kernel and declines the rest."""
    import os
    import torch
    from paper_2108_13191_b200 import _build
    if not os.path.exists(_build.FASTBIND_SO):
        pytest.skip("fastbind not built (the ctypes path is used)")
    fb = g._load_fastbind()
    assert fb is not None
    for acc in ("f32", "f16"):
        A, B, C = synth.problem(520, 384, 264, acc, seed=4)
        dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
        c1, c2 = torch.from_numpy(C.copy()).cuda(), torch.from_numpy(C.copy()).cuda()
        assert fb.gemm_default(dA, dB, c1) == 0
        g.gemm_f16(dA, dB, c2, config="auto")
        torch.cuda.synchronize()
        bits = np.uint32 if acc == "f32" else np.uint16
        assert np.array_equal(c1.cpu().numpy().view(bits), c2.cpu().numpy().view(bits))
    A = torch.zeros((64, 32), dtype=torch.float16, device="cuda")
    B = torch.zeros((32, 48), dtype=torch.float16, device="cuda")
    C = torch.zeros((64, 48), dtype=torch.float32, device="cuda")
    for a, b, c in [(A.cpu(), B, C), (A.bfloat16(), B, C), (A, B, C.double()), (A, B[:16], C),
                    (A.t().contiguous().t(), B, C), (A[:1], B, C[:1])]:
        assert fb.gemm_default(a, b, c) == -1
    # a leading dimension the library rejects comes back as its status (GEMM_ERR_INVALID_VALUE)
    assert fb.gemm_default(A[:1].expand(64, 32), B, C) == 1


@pytest.mark.parametrize("acc", ["f32", "f16"])
def test_fastbind_options_match_the_general_path(g, acc):
    """The extension's option entry (configuration, beta = 0, ReLU, bias, BF16 inputs) launches
    the same kernels as the ctypes path of gemm_f16_ex: bitwise equal results."""
    import os
    import torch
    from paper_2108_13191_b200 import _build
    if not os.path.exists(_build.FASTBIND_SO):
        pytest.skip("fastbind not built (the ctypes path is used)")
    fb = g._load_fastbind()
    M, N, K = 520, 384, 264
    A, B, C = synth.problem(M, N, K, acc, seed=6)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    bias = torch.from_numpy(synth.uniform_f32(6, 3, 1, N)[0]).cuda()
    cases = [dict(config=g.CONFIGS["solo_128x128"], beta0=0, relu=0, bias=None),
             dict(config=0, beta0=1, relu=0, bias=None),
             dict(config=0, beta0=0, relu=1, bias=bias),
             dict(config=g.CONFIGS["pair_256x256"], beta0=0, relu=0, bias=bias)]
    for bf16 in (False, True):
        a, b = (dA.bfloat16(), dB.bfloat16()) if bf16 else (dA, dB)
        for cs in cases:
            c1, c2 = torch.from_numpy(C.copy()).cuda(), torch.from_numpy(C.copy()).cuda()
            assert fb.gemm_options(a, b, c1, cs["config"], cs["beta0"], cs["relu"], cs["bias"]) == 0
            # the ctypes path: gemm_f16_ex with the same options (a non-default knob value of 0 forces it)
            g.gemm_f16(a, b, c2, config=cs["config"], beta=1 - cs["beta0"], relu=bool(cs["relu"]), bias=cs["bias"],
                       stream=torch.cuda.current_stream())
            torch.cuda.synchronize()
            bits = np.uint32 if acc == "f32" else np.uint16
            assert np.array_equal(c1.cpu().numpy().view(bits), c2.cpu().numpy().view(bits)), (bf16, cs)
    # a bias of the wrong length is declined (the Python path raises ValueError)
    assert fb.gemm_options(dA, dB, torch.from_numpy(C.copy()).cuda(), 0, 0, 0, bias[:-1]) == -1
    with pytest.raises(ValueError):
        g.gemm_f16(dA, dB, torch.from_numpy(C.copy()).cuda(), bias=bias[:-1])

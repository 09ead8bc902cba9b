"""DIAGNOSTIC ONLY: rel-Frobenius error vs K for our F32 mode and for cuBLAS
(torch.mm fp16 -> fp32 output, never on the measured path), sampled rows vs oracle."""
import os, sys, json
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch
import oracle, synth
import paper_2108_13191_b200 as g
M = N = 2048
for K in (1024, 4096, 8192, 10240, 16384, 32768):
    A, B, C = synth.problem(M, N, K, "f32", seed=0)
    C0 = np.zeros_like(C)
    rows = np.arange(0, M, 32)
    ex, _ = oracle.gemm(A, B, C0, rows=rows)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    dC = torch.zeros((M, N), dtype=torch.float32, device="cuda")
    g.gemm_f16(dA, dB, dC)
    ours = dC[torch.from_numpy(rows).cuda()].cpu().numpy().astype(np.float64)
    try:
        cub = torch.mm(dA, dB, out_dtype=torch.float32)[torch.from_numpy(rows).cuda()].cpu().numpy().astype(np.float64)
    except Exception as e:
        cub = None
    def st(x):
        if x is None: return None
        e = x - ex
        return {"rel_fro": float(np.linalg.norm(e) / np.linalg.norm(ex)), "mean_err_over_rms": float(e.mean() / np.sqrt((ex**2).mean())),
                "shrink": float(-(e * np.sign(ex)).mean() / np.sqrt((ex**2).mean()))}
    print(json.dumps({"K": K, "ours": st(ours), "cublas_fp32out": st(cub)}), flush=True)

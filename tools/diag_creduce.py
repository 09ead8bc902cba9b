"""DIAGNOSTIC: where TMA reduce-add (c_reduce) and the staged epilogue differ bitwise."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch
import paper_2108_13191_b200 as g
from parity import Guarded, device_problem
M, N, K = 777, 1000, 1000
A, B, C, gA, gB, gC = device_problem(M, N, K, "f32", seed=13, pad=(8, 8, 4))
C = C.copy()
C[::7, ::5] = -0.0
C[3, :8] = [np.inf, -np.inf, np.nan, 1e-40, -1e-40, 3.4e38, -3.4e38, 0.0]
base = Guarded(C, gC.ld)
outs = []
for red in (1, -1):
    gC.full.copy_(torch.from_numpy(base.full_host.copy()))
    g.gemm_f16(gA.view, gB.view, gC.view, config="pair_256x256_s5", c_reduce=red)
    torch.cuda.synchronize()
    outs.append(gC.result().copy())
a, b = outs[0].view(np.uint32), outs[1].view(np.uint32)
d = np.argwhere(a != b)
print("differences:", len(d))
acc = (A.astype(np.float32) @ B.astype(np.float32))
for (i, j) in d[:20]:
    print(i, j, "C_in", C[i, j], hex(C[i, j:j+1].view(np.uint32)[0]), "reduce", outs[0][i, j], hex(a[i, j]), "staged", outs[1][i, j], hex(b[i, j]), "acc~", acc[i, j])

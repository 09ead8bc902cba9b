"""DIAGNOSTIC ONLY: cuBLAS fp16 addmm at n^3 for an ncu comparison capture."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch, synth
n = 8192
A = torch.from_numpy(synth.uniform_f16(0, 0, n, n)).cuda()
B = torch.from_numpy(synth.uniform_f16(0, 1, n, n)).cuda()
C = torch.from_numpy(synth.uniform_f16(0, 2, n, n)).cuda()
O = torch.empty_like(C)
for _ in range(4):
    torch.addmm(C, A, B, out=O)
torch.cuda.synchronize()

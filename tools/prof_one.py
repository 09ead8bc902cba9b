"""Minimal driver for ncu captures: W warm-up launches then one launch per mode."""
import argparse, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import synth
import paper_2108_13191_b200 as g

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=8192)
ap.add_argument("--m", type=int, default=0)
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--k", type=int, default=0)
ap.add_argument("--modes", default="f32,f16")
ap.add_argument("--config", default="auto")
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
M = a.m or a.size; N = a.n or a.size; K = a.k or a.size
A = torch.from_numpy(synth.uniform_f16(0, 0, M, K)).cuda()
B = torch.from_numpy(synth.uniform_f16(0, 1, K, N)).cuda()
for m in a.modes.split(","):
    C = torch.from_numpy((synth.uniform_f32 if m == "f32" else synth.uniform_f16)(0, 2, M, N)).cuda()
    for _ in range(a.warmup + a.reps):
        g.gemm_f16(A, B, C, config=a.config)
    torch.cuda.synchronize()
print("done")

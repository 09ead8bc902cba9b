"""One launch (after 2 warm-ups) of a variant, for ncu metric passes. Args: JSON kwargs."""
import os, sys, json
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch, synth
import paper_2108_13191_b200 as g
v = json.loads(sys.argv[1]) if len(sys.argv) > 1 else {}
M = int(v.pop("M", 8192)); N = int(v.pop("N", M)); K = int(v.pop("K", M)); mode = v.pop("mode", "f32")
A = torch.from_numpy(synth.uniform_f16(0, 0, M, K)).cuda()
B = torch.from_numpy(synth.uniform_f16(0, 1, K, N)).cuda()
C = torch.from_numpy((synth.uniform_f32 if mode == "f32" else synth.uniform_f16)(0, 2, M, N)).cuda()
for _ in range(3): g.gemm_f16(A, B, C, **v)
torch.cuda.synchronize()

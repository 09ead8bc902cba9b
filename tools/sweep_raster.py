"""Ablation: raster group height (tiles) vs time at n^3, back-to-back launches."""
import os, sys, json
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch, synth
import paper_2108_13191_b200 as g
n = int(os.environ.get("N", "8192"))
mode = os.environ.get("MODE", "f32")
groups = [int(x) for x in os.environ.get("GROUPS", "1,2,4,8,16,32").split(",")]
A = torch.from_numpy(synth.uniform_f16(0, 0, n, n)).cuda()
B = torch.from_numpy(synth.uniform_f16(0, 1, n, n)).cuda()
C = torch.from_numpy((synth.uniform_f32 if mode == "f32" else synth.uniform_f16)(0, 2, n, n)).cuda()
for gm in groups:
    for _ in range(5): g.gemm_f16(A, B, C, group_m=gm)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(20): g.gemm_f16(A, B, C, group_m=gm)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 20
    print(json.dumps({"mode": mode, "group_m": gm, "ms": round(ms, 4), "tflops": round(2 * n**3 / ms / 1e9, 1)}), flush=True)

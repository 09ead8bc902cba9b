"""DIAGNOSTIC: phase timeline of CTA 0 of a split-K cluster kernel (globaltimer ns)."""
import os, sys, json
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch, synth
import paper_2108_13191_b200 as g
for spec in sys.argv[1:]:
    shape, mode, cfg = spec.split(":")
    kw = {}
    M, N, K = (int(x) for x in shape.split("x"))
    A = torch.from_numpy(synth.uniform_f16(0, 0, M, K)).cuda()
    B = torch.from_numpy(synth.uniform_f16(0, 1, K, N)).cuda()
    C = torch.from_numpy((synth.uniform_f32 if mode == "f32" else synth.uniform_f16)(0, 2, M, N)).cuda()
    tr = torch.zeros(512, dtype=torch.int64, device="cuda")
    for _ in range(3): g.gemm_f16(A, B, C, config=cfg)
    g.gemm_f16(A, B, C, config=cfg, trace=tr, **kw)
    torch.cuda.synchronize()
    t = tr.cpu().numpy()[:8]
    names = ["entry", "setup", "acc_ready", "all_mainloops_done", "pushed", "recv_in", "exit", "reduced"]
    print(spec, " ".join(f"{n}={(x - t[0]) / 1000:.2f}us" for n, x in zip(names, t)))

#!/bin/bash
python - <<'PY'
import sys; sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np, torch, oracle, synth
import paper_2108_13191_b200 as g
from parity import check
for acc in ("f32", "f16"):
    for (M, N, K) in [(1024, 1024, 1024), (300, 520, 777), (1024, 1024, 2048)]:
        A, B, C = synth.problem(M, N, K, acc, seed=3)
        dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
        pad = lambda x: x
        dC = torch.from_numpy(C.copy()).cuda() if (N * (4 if acc == "f32" else 2)) % 16 == 0 else None
        if dC is None: continue
        if (K * 2) % 16: continue
        g.gemm_f16(dA, dB, dC, config="splitk_128x128_s2"); torch.cuda.synchronize()
        ex, _ = oracle.gemm(A, B, C)
        print(acc, (M, N, K), check(dC.cpu().numpy(), ex, A, B, acc, K, "s2_128")["rel_fro"])
PY
SHAPES=1024x1024x1024,1024x1024x2048,512x2048x1024,2048x512x2048 CFGS=0,5,12,15 timeout 600 python tools/graph_bench.py

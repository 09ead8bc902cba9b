import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, torch
import paper_2108_13191_b200 as g
from parity import device_problem
for acc in ("f32", "f16"):
    for (M, N, K) in [(1, 1, 1), (1, 8, 1), (2, 3, 64), (7, 9, 15), (33, 40, 17), (40, 1, 40), (17, 24, 65), (1, 100, 8), (5, 1, 8)]:
        for cfg in ("auto", "pair_256x256", "solo_128x64"):
            A, B, C, gA, gB, gC = device_problem(M, N, K, acc, seed=1, pad=(8, 8, 8))
            g.gemm_f16(gA.view, gB.view, gC.view, config=cfg)
            torch.cuda.synchronize()
            now = gC.full.cpu().numpy()
            a = now.view(np.uint32 if now.dtype.itemsize == 4 else np.uint16)
            b = gC.full_host.view(a.dtype)
            mask = np.ones(now.shape, bool); mask[:M, :N] = False
            bad = np.argwhere((a != b) & mask)
            print(acc, (M, N, K), cfg, "ldc", gC.ld, "shape", now.shape, "bad", len(bad), bad[:6].tolist(),
                  [hex(int(a[tuple(x)])) for x in bad[:3]], [float(now[tuple(x)]) for x in bad[:3]])

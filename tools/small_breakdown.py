"""DIAGNOSTIC: where a small GEMM's time goes: per-GEMM time in CUDA-graph replay vs
the kernel body seen by CTA 0 (globaltimer trace) vs a trivial-kernel graph floor."""
import os, sys, json, statistics
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch, synth
import paper_2108_13191_b200 as g

def graph_us(fn, R=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3): fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        for _ in range(R): fn()
    gr.replay(); torch.cuda.synchronize()
    ts = []
    for _ in range(7):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); gr.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / R * 1000)
    return statistics.median(ts)

x = torch.zeros(16, device="cuda")
print(json.dumps({"trivial_kernel_graph_us": round(graph_us(lambda: x.add_(1)), 2)}))
for (M, N, K, mode, cfg) in ((1024, 1024, 1024, "f16", "solo_128x64"), (1024, 1024, 1024, "f32", "solo_128x64"),
                             (256, 256, 256, "f32", "solo_128x64"), (2048, 2048, 2048, "f16", "pair_256x256_k128")):
    A = torch.from_numpy(synth.uniform_f16(0, 0, M, K)).cuda()
    B = torch.from_numpy(synth.uniform_f16(0, 1, K, N)).cuda()
    C = torch.from_numpy((synth.uniform_f32 if mode == "f32" else synth.uniform_f16)(0, 2, M, N)).cuda()
    us = graph_us(lambda: g.gemm_f16(A, B, C, config=cfg))
    tr = torch.zeros(512, dtype=torch.int64, device="cuda")
    bodies = []
    for _ in range(5):
        tr.zero_()
        g.gemm_f16(A, B, C, config=cfg, trace=tr); torch.cuda.synchronize()
        t = tr.cpu().numpy().reshape(64, 8)
        bodies.append({"entry_to_setup": (t[62, 1] - t[62, 0]) / 1000, "setup_to_mma0": (t[0, 0] - t[62, 1]) / 1000,
                       "mma_span": (t[0, 2] - t[0, 0]) / 1000, "mma_end_to_stored": (t[0, 6] - t[0, 2]) / 1000,
                       "stored_to_exit": (t[62, 2] - t[0, 6]) / 1000, "entry_to_exit": (t[62, 2] - t[62, 0]) / 1000})
    med = {k: round(statistics.median(b[k] for b in bodies), 2) for k in bodies[0]}
    print(json.dumps({"shape": [M, N, K], "mode": mode, "config": cfg, "graph_us_per_gemm": round(us, 2), "cta0_us": med}), flush=True)

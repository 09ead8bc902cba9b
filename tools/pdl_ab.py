"""A/B: programmatic dependent launch (pdl=1) vs off, per-GEMM time for chains of
dependent GEMMs (C accumulates in place), in CUDA-graph replay and back-to-back
stream launches; interleaved rounds, medians."""
import os, sys, json, statistics
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch, synth
import paper_2108_13191_b200 as g

def make_graph(fn, R):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3): fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        for _ in range(R): fn()
    gr.replay(); torch.cuda.synchronize()
    return gr

def time_graph(gr, R):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); gr.replay(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / R * 1000

def time_stream(fn, R):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(R): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / R * 1000

for (M, N, K, mode, R) in ((256, 256, 256, "f32", 50), (1024, 1024, 1024, "f16", 50), (1024, 1024, 1024, "f32", 50),
                           (2048, 2048, 2048, "f16", 30), (4096, 1024, 1024, "f32", 30), (8192, 8192, 8192, "f16", 5)):
    A = torch.from_numpy(synth.uniform_f16(0, 0, M, K)).cuda()
    B = torch.from_numpy(synth.uniform_f16(0, 1, K, N)).cuda()
    C = torch.from_numpy((synth.uniform_f32 if mode == "f32" else synth.uniform_f16)(0, 2, M, N)).cuda()
    fns = {p: (lambda p=p: g.gemm_f16(A, B, C, pdl=p)) for p in (-1, 1)}
    graphs = {p: make_graph(fns[p], R) for p in fns}
    res = {f"{kind}_pdl{p}": [] for kind in ("graph", "stream") for p in fns}
    for _ in range(7):
        for p in fns:
            res[f"graph_pdl{p}"].append(time_graph(graphs[p], R))
            res[f"stream_pdl{p}"].append(time_stream(fns[p], R))
    print(json.dumps({"shape": [M, N, K], "mode": mode, **{k: round(statistics.median(v), 2) for k, v in res.items()}}), flush=True)

"""CUDA-graph-replay A/B of library builds (GPU-only time per GEMM): LIBS=a.so,b.so SHAPES=MxNxK,... MODES=f32,f16.
The default build is the baseline; every build is captured once per shape and replayed in a shuffled order, median of 9."""
import os, sys, json, statistics, random
sys.path.insert(0, os.getcwd())
import torch, synth
import paper_2108_13191_b200 as g
libs = [None] + [l for l in os.environ.get("LIBS", "").split(",") if l]
handles = {None: g.load_library()}
for l in libs[1:]:
    g._lib = None; g._build.LIB = os.path.abspath(l); handles[l] = g.load_library(build_if_missing=False)
shapes = [tuple(int(x) for x in t.split("x")) for t in os.environ["SHAPES"].split(",")]
R = 20
for (M, N, K) in shapes:
    for mode in os.environ.get("MODES", "f32,f16").split(","):
        A = torch.from_numpy(synth.uniform_f16(0, 0, M, K)).cuda(); B = torch.from_numpy(synth.uniform_f16(0, 1, K, N)).cuda()
        C = torch.from_numpy((synth.uniform_f32 if mode == "f32" else synth.uniform_f16)(0, 2, M, N)).cuda()
        graphs = {}
        for l in libs:
            g._lib = handles[l]
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(3): g.gemm_f16(A, B, C, stream=s)
            torch.cuda.synchronize()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=s):
                for _ in range(R): g.gemm_f16(A, B, C, stream=s)
            graphs[l] = (gr, s)
        res = {l: [] for l in libs}
        rng = random.Random(0)
        for _ in range(9):
            order = list(libs); rng.shuffle(order)
            for l in order:
                gr, s = graphs[l]
                with torch.cuda.stream(s):
                    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                    e0.record(s); gr.replay(); e1.record(s); torch.cuda.synchronize()
                res[l].append(e0.elapsed_time(e1) / R * 1000)
        print(json.dumps({"shape": [M, N, K], "mode": mode, **{str(l): round(statistics.median(v), 3) for l, v in res.items()}}), flush=True)

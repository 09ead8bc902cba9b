"""GPU-side time per GEMM for small shapes: R launches captured in one CUDA graph
and replayed (removes host enqueue cost), per config."""
import os, sys, json, statistics
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch, synth
import paper_2108_13191_b200 as g
shapes = [tuple(int(x) for x in t.split("x")) for t in os.environ.get("SHAPES", "256x256x256,512x512x512,1024x1024x1024,2048x2048x2048,4096x1024x1024,2048x2048x512").split(",")]
CFGS = [int(c) for c in os.environ.get("CFGS", "1,2,4,5,6").split(",")]
OPTS = json.loads(os.environ.get("OPTS", "{}"))   # extra gemm_f16 keyword arguments
R = 20
for (M, N, K) in shapes:
    for mode in os.environ.get("MODES", "f32,f16").split(","):
        A = torch.from_numpy(synth.uniform_f16(0, 0, M, K)).cuda()
        B = torch.from_numpy(synth.uniform_f16(0, 1, K, N)).cuda()
        C = torch.from_numpy((synth.uniform_f32 if mode == "f32" else synth.uniform_f16)(0, 2, M, N)).cuda()
        row = {"shape": [M, N, K], "mode": mode, "auto": g.pick_config(M, N, K, 0 if mode == "f32" else 1)}
        for cfg in CFGS:
            if cfg == g.CONFIGS["pair_256x512"] and mode == "f32":
                continue   # (F16 C only)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(3): g.gemm_f16(A, B, C, config=cfg, **OPTS)
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=s):
                for _ in range(R): g.gemm_f16(A, B, C, config=cfg, **OPTS)
            graph.replay(); torch.cuda.synchronize()
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                e0.record(); graph.replay(); e1.record(); torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) / R * 1000)
            us = statistics.median(ts)
            row[f"cfg{cfg}_us"] = round(us, 2)
            row[f"cfg{cfg}_tflops"] = round(2 * M * N * K / us / 1e6, 1)
        print(json.dumps(row), flush=True)

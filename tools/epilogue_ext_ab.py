"""SHAPE=MxNxK (default 8192^3): the fused-epilogue extensions (BF16 inputs, beta = 0, bias + ReLU) against the plain
F16-input GEMM in both modes, shuffled blocks of back-to-back launches, medians."""
import json, os, sys, statistics, random
sys.path.insert(0, os.getcwd())
import torch, synth
import paper_2108_13191_b200 as g
M, N, K = (int(x) for x in os.environ.get("SHAPE", "8192x8192x8192").split("x"))
n = N
A = torch.from_numpy(synth.uniform_f16(0, 0, M, K)).cuda(); B = torch.from_numpy(synth.uniform_f16(0, 1, K, N)).cuda()
Ab, Bb = A.to(torch.bfloat16), B.to(torch.bfloat16)
Cs = {"f32": torch.from_numpy(synth.uniform_f32(0, 2, M, N)).cuda(), "f16": torch.from_numpy(synth.uniform_f16(0, 2, M, N)).cuda()}
bias = torch.from_numpy(synth.uniform_f32(0, 3, 1, N)[0]).cuda()
V = {"f32_f16in": lambda: g.gemm_f16(A, B, Cs["f32"]), "f32_bf16in": lambda: g.gemm_f16(Ab, Bb, Cs["f32"]),
     "f16_f16in": lambda: g.gemm_f16(A, B, Cs["f16"]), "f16_bf16in": lambda: g.gemm_f16(Ab, Bb, Cs["f16"]),
     "f32_beta0": lambda: g.gemm_f16(A, B, Cs["f32"], beta=0), "f32_bias_relu": lambda: g.gemm_f16(A, B, Cs["f32"], bias=bias, relu=True),
     "f16_beta0": lambda: g.gemm_f16(A, B, Cs["f16"], beta=0), "f16_bias_relu": lambda: g.gemm_f16(A, B, Cs["f16"], bias=bias, relu=True),
     "f32_bias": lambda: g.gemm_f16(A, B, Cs["f32"], bias=bias),
     "f32_bias_staged": lambda: g.gemm_f16(A, B, Cs["f32"], bias=bias, c_reduce=-1)}
for f in V.values(): f(); f()
torch.cuda.synchronize()
res = {k: [] for k in V}; rng = random.Random(0)
for _ in range(10):
    order = list(V); rng.shuffle(order)
    for k in order:
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True); e0.record()
        for _ in range(4): V[k]()
        e1.record(); torch.cuda.synchronize(); res[k].append(e0.elapsed_time(e1) / 4)
for k, v in res.items():
    ms = statistics.median(v); print(json.dumps({"shape": [M, N, K], "variant": k, "ms": round(ms, 4), "tflops": round(2 * M * N * K / ms / 1e9, 1)}))

"""A/B timing of kernel variants: round-robin blocks of back-to-back launches
(medians over rounds), so drifting power/thermal state hits every variant alike.
VARIANTS='[{"mode":"f32"}, {"mode":"f32","l2_hints":-1}]' python tools/ab.py"""
import os, sys, json, statistics
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch, synth
import paper_2108_13191_b200 as g
variants = json.loads(os.environ.get("VARIANTS", '[{"mode":"f32"}]'))
rounds = int(os.environ.get("ROUNDS", "5")); reps = int(os.environ.get("REPS", "20"))
M = int(os.environ.get("M", "8192")); N = int(os.environ.get("N", str(M))); K = int(os.environ.get("K", str(M)))
A = torch.from_numpy(synth.uniform_f16(0, 0, M, K)).cuda()
B = torch.from_numpy(synth.uniform_f16(0, 1, K, N)).cuda()
Cs = {"f32": torch.from_numpy(synth.uniform_f32(0, 2, M, N)).cuda(), "f16": torch.from_numpy(synth.uniform_f16(0, 2, M, N)).cuda()}
res = {i: [] for i in range(len(variants))}
Ab, Bb = A.bfloat16(), B.bfloat16()
bias_vec = torch.from_numpy(synth.uniform_f32(7, 3, 1, N)[0]).cuda()
def run(v):
    kw = {k: x for k, x in v.items() if k not in ("mode", "bf16", "bias")}
    if v.get("bias"):
        kw["bias"] = bias_vec
    a, b = (Ab, Bb) if v.get("bf16") else (A, B)
    g.gemm_f16(a, b, Cs[v.get("mode", "f32")], **kw)
for v in variants:
    for _ in range(3): run(v)
torch.cuda.synchronize()
for r in range(rounds):
    for i, v in enumerate(variants):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        for _ in range(reps): run(v)
        e.record(); torch.cuda.synchronize()
        res[i].append(s.elapsed_time(e) / reps)
for i, v in enumerate(variants):
    ms = statistics.median(res[i])
    print(json.dumps({"variant": v, "shape": [M, N, K], "ms_median": round(ms, 4), "tflops": round(2 * M * N * K / ms / 1e9, 1),
                      "ms_all": [round(x, 4) for x in res[i]]}), flush=True)

"""bench.py's step (one F32 GEMM, then one F16 GEMM, 8192^3, inputs larger than L2) with the F16
GEMM's configuration varied: W warm-up steps then S timed steps per block, blocks in a shuffled
order per round, medians.  F16CFGS='auto,pair_256x256' STEPS=20 ROUNDS=10 python tools/step_ab.py"""
import os, sys, json, random, statistics
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch, synth
import paper_2108_13191_b200 as g
n = int(os.environ.get("N", "8192"))
cfgs = os.environ.get("F16CFGS", "auto,pair_256x256").split(",")
steps = int(os.environ.get("STEPS", "20")); warm = int(os.environ.get("WARM", "3")); rounds = int(os.environ.get("ROUNDS", "10"))
A = torch.from_numpy(synth.uniform_f16(0, 0, n, n)).cuda()
B = torch.from_numpy(synth.uniform_f16(0, 1, n, n)).cuda()
C32 = torch.from_numpy(synth.uniform_f32(0, 2, n, n)).cuda()
C16 = torch.from_numpy(synth.uniform_f16(0, 2, n, n)).cuda()
def step(cfg):
    g.gemm_f16(A, B, C32)
    g.gemm_f16(A, B, C16, config=cfg)
res = {c: [] for c in cfgs}
rng = random.Random(1)
for r in range(rounds):
    order = list(cfgs); rng.shuffle(order)
    for c in order:
        for _ in range(warm): step(c)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(steps): step(c)
        e1.record(); torch.cuda.synchronize()
        res[c].append(e0.elapsed_time(e1) / steps)
for c in cfgs:
    ms = statistics.median(res[c])
    print(json.dumps({"f16_config": c, "steps": steps, "ms_per_step_median": round(ms, 4),
                      "tflops_step": round(2 * 2 * n ** 3 / ms / 1e9, 1), "all": [round(x, 4) for x in res[c]]}), flush=True)

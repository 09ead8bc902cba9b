"""A/B of option sets AND library builds in one process (blocks of back-to-back launches in a
shuffled order per round, medians): VARIANTS='[{"mode":"f32","config":"pair_256x512"},
{"lib":"scratch/libA.so","mode":"f32","config":"pair_256x512","promote_k":-1}]'.
A variant's "lib" swaps the binding's library handle (same ABI, another build)."""
import ctypes, json, os, statistics, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch, synth
import paper_2108_13191_b200 as g
variants = json.loads(os.environ["VARIANTS"])
rounds = int(os.environ.get("ROUNDS", "5")); reps = int(os.environ.get("REPS", "20"))
M = int(os.environ.get("M", "8192")); N = int(os.environ.get("N", str(M))); K = int(os.environ.get("K", str(M)))
base = g.load_library()
handles = {None: base}
for v in variants:
    if v.get("lib") and v["lib"] not in handles:
        g._lib = None
        g._build.LIB = os.path.abspath(v["lib"])
        handles[v["lib"]] = g.load_library(build_if_missing=False)
A = torch.from_numpy(synth.uniform_f16(0, 0, M, K)).cuda()
B = torch.from_numpy(synth.uniform_f16(0, 1, K, N)).cuda()
Cs = {"f32": torch.from_numpy(synth.uniform_f32(0, 2, M, N)).cuda(), "f16": torch.from_numpy(synth.uniform_f16(0, 2, M, N)).cuda()}
def run(v):
    g._lib = handles[v.get("lib")]
    kw = {k: x for k, x in v.items() if k not in ("mode", "lib")}
    g.gemm_f16(A, B, Cs[v.get("mode", "f32")], **kw)
for v in variants:
    for _ in range(3): run(v)
torch.cuda.synchronize()
res = {i: [] for i in range(len(variants))}
import random
rng = random.Random(0)
for r in range(rounds):
    # shuffled order per round: under the power cap the variant right after the round's
    # Python gap runs on a cooler board (a fixed order favoured variant 0 by up to ~4 %)
    order = list(range(len(variants)))
    rng.shuffle(order)
    for i in order:
        v = variants[i]
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        for _ in range(reps): run(v)
        e.record(); torch.cuda.synchronize()
        res[i].append(s.elapsed_time(e) / reps)
for i, v in enumerate(variants):
    ms = statistics.median(res[i])
    print(json.dumps({"variant": v, "shape": [M, N, K], "ms_median": round(ms, 4), "tflops": round(2 * M * N * K / ms / 1e9, 1),
                      "ms_all": [round(x, 4) for x in res[i]]}), flush=True)

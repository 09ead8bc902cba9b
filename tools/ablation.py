"""B200 analogue of the paper's incremental-optimisation study (fig:gradual-opts,
PAPER.md P:951-965) at M=N=K=8192, F32 accumulate: the same kernel with design
choices switched on one at a time (cumulative), plus one-at-a-time removals from
the full design.  Timing: round-robin blocks of back-to-back launches (CUDA
events), median over rounds, all variants in one process on one GPU."""
import os, sys, json, statistics
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch, synth
import paper_2108_13191_b200 as g

n = int(os.environ.get("N", "8192"))
mode = os.environ.get("MODE", "f32")
rounds = int(os.environ.get("ROUNDS", "12")); reps = int(os.environ.get("REPS", "4"))
import random
rng = random.Random(0)
naive = dict(config="solo_128x256", ring_stages=1, acc_bufs=1, group_m=1, l2_hints=-1, promote_k=-1)
cumulative = [
    ("naive: 1-CTA 128x256, 1-stage ring, single TMEM acc, row-major order", dict(naive)),
    ("+ 4-stage TMA/mbarrier ring", dict(naive, ring_stages=0)),
    ("+ double-buffered TMEM (epilogue overlaps MMA)", dict(naive, ring_stages=0, acc_bufs=0)),
    ("+ 2-CTA pair 256x256 (cta_group::2), 6 stages", dict(naive, config="pair_256x256", ring_stages=0, acc_bufs=0)),
    ("+ grouped raster (group_m=8)", dict(naive, config="pair_256x256", ring_stages=0, acc_bufs=0, group_m=0)),
    ("+ L2 eviction hints", dict(naive, config="pair_256x256", ring_stages=0, acc_bufs=0, group_m=0, l2_hints=0)),
    ("+ K-chunk promotion to F32 registers (accuracy)", dict(config="pair_256x256")),
    ("+ 128-deep K stages (= shipped default)", dict()),
]
removals = [
    ("full (shipped default), again", dict()),
    ("full - ring (1 x 128-deep stage)", dict(ring_stages=1)),
    ("full - ring (2 x 128-deep stages)", dict(ring_stages=2)),
    ("full - TMEM double buffer", dict(acc_bufs=1)),
    ("full - persistence (one cluster per tile)", dict(max_clusters=100000)),
    ("full - 2-CTA (1-CTA 128x256, 64-deep)", dict(config="solo_128x256")),
    ("full - 128-deep stages (64-deep, 6 stages)", dict(config="pair_256x256")),
    ("full - raster (row-major tiles)", dict(group_m=1)),
    ("full - L2 hints", dict(l2_hints=-1)),
    ("full - promotion", dict(promote_k=-1)),
    ("full - 128-deep stages - swizzle (no-swizzle UMMA layout, 16-byte TMA boxes, unswizzled epilogue staging)",
     dict(config="pair_256x256", swizzle=-1)),
    ("full - warp specialisation (1 thread pipelines TMA + MMA, 128x128 per CTA, epilogue after the mainloop)",
     dict(warp_specialize=-1)),
    ("full - warp specialisation, 1-stage pipeline (the paper's single stage)", dict(warp_specialize=-1, ring_stages=1)),
]
variants = cumulative + removals
A = torch.from_numpy(synth.uniform_f16(0, 0, n, n)).cuda()
B = torch.from_numpy(synth.uniform_f16(0, 1, n, n)).cuda()
C = torch.from_numpy((synth.uniform_f32 if mode == "f32" else synth.uniform_f16)(0, 2, n, n)).cuda()
res = {i: [] for i in range(len(variants))}
for name, kw in variants:
    g.gemm_f16(A, B, C, **kw)
torch.cuda.synchronize()
for r in range(rounds):
    order = list(range(len(variants)))
    rng.shuffle(order)   # no variant always runs in the same (thermal) position of a round
    for i in order:
        name, kw = variants[i]
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        for _ in range(reps): g.gemm_f16(A, B, C, **kw)
        e.record(); torch.cuda.synchronize()
        res[i].append(s.elapsed_time(e) / reps)
for i, (name, kw) in enumerate(variants):
    ms = statistics.median(res[i])
    print(json.dumps({"variant": name, "kwargs": kw, "n": n, "mode": mode, "ms": round(ms, 4),
                      "ms_p25": round(sorted(res[i])[len(res[i]) // 4], 4), "ms_p75": round(sorted(res[i])[3 * len(res[i]) // 4], 4),
                      "tflops": round(2 * n ** 3 / ms / 1e9, 1), "group": "cumulative" if i < len(cumulative) else "removal"}), flush=True)

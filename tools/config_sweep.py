"""Per-size 'best performing version' on the square sweep: for each size,
the auto pick and the candidate configurations run in one process, shuffled blocks of
back-to-back launches per round, medians.  JSON lines: shape, mode, auto config, ms per config.
usage: LO=1024 HI=8192 STEP=256 python tools/config_sweep.py"""
import json, os, random, statistics, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch, synth
import paper_2108_13191_b200 as g

lo, hi, step = int(os.environ.get("LO", "1024")), int(os.environ.get("HI", "8192")), int(os.environ.get("STEP", "256"))
rounds = int(os.environ.get("ROUNDS", "5"))
CANDS = {"f32": ["auto", "pair_256x256", "pair_256x256_k128", "pair_256x256_s4", "pair_256x256_s5", "solo_128x128"],
         "f16": ["auto", "pair_256x256", "pair_256x256_k128", "pair_256x256_s4", "pair_256x256_s5", "pair_256x512",
                 "solo_128x128"]}
Abig = torch.from_numpy(synth.uniform_f16(0, 0, hi, hi)).cuda()
Bbig = torch.from_numpy(synth.uniform_f16(0, 1, hi, hi)).cuda()
rng = random.Random(0)
for n in range(lo, hi + 1, step):
    A, B = Abig[:n, :n].contiguous(), Bbig[:n, :n].contiguous()
    reps = max(3, min(40, int(2e12 / (2.0 * n ** 3))))
    for mode in ("f32", "f16"):
        C = torch.from_numpy((synth.uniform_f32 if mode == "f32" else synth.uniform_f16)(0, 2, n, n)).cuda()
        cands = CANDS[mode]
        for c in cands:
            for _ in range(2):
                g.gemm_f16(A, B, C, config=c)
        torch.cuda.synchronize()
        res = {c: [] for c in cands}
        for _ in range(rounds):
            order = list(cands)
            rng.shuffle(order)
            for c in order:
                e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                e0.record()
                for _ in range(reps):
                    g.gemm_f16(A, B, C, config=c)
                e1.record()
                torch.cuda.synchronize()
                res[c].append(e0.elapsed_time(e1) / reps)
        ms = {c: round(statistics.median(v), 5) for c, v in res.items()}
        best = min(ms, key=ms.get)
        print(json.dumps({"n": n, "mode": mode, "auto_config": g.pick_config(n, n, n, 0 if mode == "f32" else 1),
                          "ms": ms, "best": best, "auto_over_best": round(ms["auto"] / ms[best], 4)}), flush=True)
        del C

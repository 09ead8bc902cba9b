"""Kernel-side cost of the fused N-shard GEMM + all-gather (gemm_f16_gather) on ONE
GPU: one rank's slab of the 16384^3 problem at P ranks (16384 x 16384/P x 16384), timed as the
plain slab GEMM and as the fused kernel storing every finished tile into P-1 extra C buffers.
With one GPU the "peers" are buffers on the same device, so the extra stores go to local HBM
instead of NVLink; the numbers bound the epilogue-side overhead of the fused path, not the
link.  Interleaved rounds (shuffled), CUDA events, median.  JSON lines on stdout."""
import json, os, random, statistics, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch, synth
import paper_2108_13191_b200 as g

n = int(os.environ.get("N", "16384"))
rounds, reps = int(os.environ.get("ROUNDS", "5")), int(os.environ.get("REPS", "3"))
for P in (int(x) for x in os.environ.get("RANKS", "2,4,8").split(",")):
    nr = n // P
    A = torch.from_numpy(synth.uniform_f16(0, 0, n, n)).cuda()
    B = torch.from_numpy(synth.uniform_f16(0, 1, n, n, col_lo=0, col_hi=nr)).cuda()
    for mode in os.environ.get("MODES", "f32,f16").split(","):
        dt = torch.float32 if mode == "f32" else torch.float16
        Cs = torch.zeros((n, nr), dtype=dt, device="cuda")     # plain: this rank's slab only
        Cf = torch.zeros((n, n), dtype=dt, device="cuda")      # fused: full C, this rank's columns
        peers = [torch.zeros((n, n), dtype=dt, device="cuda") for _ in range(P - 1)]
        variants = {"plain": lambda: g.gemm_f16(A, B, Cs),
                    "fused": lambda: g.gemm_f16_gather(A, B, Cf, 0, peers=peers)}
        for f in variants.values():
            f()
        torch.cuda.synchronize()
        res = {k: [] for k in variants}
        rng = random.Random(0)
        for _ in range(rounds):
            order = list(variants)
            rng.shuffle(order)
            for k in order:
                e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                e0.record()
                for _ in range(reps):
                    variants[k]()
                e1.record()
                torch.cuda.synchronize()
                res[k].append(e0.elapsed_time(e1) / reps)
        ms = {k: statistics.median(v) for k, v in res.items()}
        print(json.dumps({"P": P, "mode": mode, "slab": [n, nr, n], "plain_ms": round(ms["plain"], 4),
                          "fused_ms": round(ms["fused"], 4), "fused_over_plain": round(ms["fused"] / ms["plain"], 4),
                          "extra_bytes_stored_per_rank": (P - 1) * n * nr * Cf.element_size()}), flush=True)
        del Cs, Cf, peers
        torch.cuda.empty_cache()
    del A, B

"""EXPERIMENT (DESIGN R16): the tensor core's binary16 accumulation
(idesc c_format = F16, `accum_f16=True`).  Diagnostic only, never the default path.
1. decoding: ones x ones;  2. rounding probe (P4 analogue, ulp(1) = 2^-10);
3. rel-Frobenius error vs K against the oracle for several promotion intervals;
4. speed vs the F32-accumulating default (interleaved rounds)."""
import os, sys, json, statistics
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch
import oracle, synth
import paper_2108_13191_b200 as g

def run(A, B, C, **kw):
    dA, dB, dC = (torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (A, B, C))
    g.gemm_f16(dA, dB, dC, **kw); torch.cuda.synchronize()
    return dC.cpu().numpy()

# 1. decoding
for cfg in ("solo_128x64", "pair_256x256", "pair_256x256_k128"):
    for K in (16, 64, 1000):
        A = np.ones((256, K), np.float16); B = np.ones((K, 256), np.float16)
        out = run(A, B, np.zeros((256, 256), np.float32), accum_f16=True, config=cfg, promote_k=-1)
        print(json.dumps({"probe": "ones", "config": cfg, "K": K, "min": float(out.min()), "max": float(out.max())}))

# 2. rounding probe: exact 1 + 3*2^-12 = 1 + 0.75 ulp_f16(1)
def probe(split, sign):
    K = 32
    A = np.zeros((128, K), np.float16); B = np.zeros((K, 128), np.float16)
    A[0, 0] = sign; B[0, 0] = 1
    ks = [16, 17, 18] if split else [1, 2, 3]
    for k in ks:
        A[0, k] = sign * 2.0 ** -6; B[k, 0] = 2.0 ** -6
    out = run(A, B, np.zeros((128, 128), np.float32), accum_f16=True, config="solo_128x64", promote_k=-1)
    v = float(out[0, 0]); one_up = sign * (1 + 2.0 ** -10)
    return {"probe": "round", "k16_blocks": "separate" if split else "same", "sign": sign, "value": v,
            "reading": "RNE/up" if v == one_up else ("RZ/trunc" if v == sign * 1.0 else "other")}
for split in (True, False):
    for sign in (1.0, -1.0):
        print(json.dumps(probe(split, sign)))
# half-ulp tie: 1 + 2*2^-12 = 1 + 0.5 ulp -> RNE gives 1 (even)
A = np.zeros((128, 32), np.float16); B = np.zeros((32, 128), np.float16)
A[0, 0] = 1; B[0, 0] = 1; A[0, 16] = A[0, 17] = 2.0 ** -6; B[16, 0] = B[17, 0] = 2.0 ** -6
print(json.dumps({"probe": "tie 1+0.5ulp", "value": float(run(A, B, np.zeros((128, 128), np.float32), accum_f16=True,
                                                             config="solo_128x64", promote_k=-1)[0, 0])}))

# 3. error vs K (F16 output mode, C_in random and C_in = 0), sampled rows
M = N = 1024
for K in (1024, 4096, 8192, 16384):
    A, B, C = synth.problem(M, N, K, "f16", seed=0)
    rows = np.arange(0, M, 16)
    for cin in ("random", "zero"):
        Cx = C if cin == "random" else np.zeros_like(C)
        ex, _ = oracle.gemm(A, B, Cx, rows=rows)
        rec = {"K": K, "C_in": cin}
        for name, kw in (("f32acc_default", {}), ("f16acc_one_chain", {"accum_f16": True, "promote_k": -1}),
                         ("f16acc_promote2048", {"accum_f16": True}),
                         ("f16acc_promote512", {"accum_f16": True, "promote_k": 512, "config": "pair_256x256"}),
                         ("f16acc_promote256", {"accum_f16": True, "promote_k": 256, "config": "pair_256x256"})):
            out = run(A, B, Cx, **kw)[rows].astype(np.float64)
            e = out - ex
            rec[name] = {"rel_fro": float(np.linalg.norm(e) / np.linalg.norm(ex)),
                         "bias_over_rms": float(e.mean() / np.sqrt((ex ** 2).mean())), "finite": bool(np.isfinite(out).all())}
        print(json.dumps(rec), flush=True)

# 4. speed (interleaved rounds, 8192^3)
M = N = K = 8192
A = torch.from_numpy(synth.uniform_f16(0, 0, M, K)).cuda(); B = torch.from_numpy(synth.uniform_f16(0, 1, K, N)).cuda()
Cs = {"f32": torch.from_numpy(synth.uniform_f32(0, 2, M, N)).cuda(), "f16": torch.from_numpy(synth.uniform_f16(0, 2, M, N)).cuda()}
variants = [("f16", {}), ("f16", {"accum_f16": True}), ("f16", {"accum_f16": True, "promote_k": -1}),
            ("f32", {}), ("f32", {"accum_f16": True})]
res = {i: [] for i in range(len(variants))}
for mode, kw in variants:
    for _ in range(3): g.gemm_f16(A, B, Cs[mode], **kw)
torch.cuda.synchronize()
for r in range(7):
    for i, (mode, kw) in enumerate(variants):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        for _ in range(10): g.gemm_f16(A, B, Cs[mode], **kw)
        e.record(); torch.cuda.synchronize()
        res[i].append(s.elapsed_time(e) / 10)
for i, (mode, kw) in enumerate(variants):
    ms = statistics.median(res[i])
    print(json.dumps({"speed": mode, "kw": kw, "ms": round(ms, 4), "tflops": round(2 * M * N * K / ms / 1e9, 1)}))

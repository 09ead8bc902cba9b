"""EXPERIMENT: is the tensor core's binary16 accumulation bit-exactly
acc <- RNE16(acc + exact sum of the 16 products of one k16 instruction)?
Host emulation in float64 (products of binary16 values and sums of 16 of them are
exact in float64 for these inputs), compared bitwise with accum_f16, promote_k=-1,
C_in = 0, F32 output (which holds the binary16 accumulator exactly)."""
import os, sys, json
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch
import synth
import paper_2108_13191_b200 as g

def emulate(A, B, block=16):
    A64, B64 = A.astype(np.float64), B.astype(np.float64)
    acc = np.zeros((A.shape[0], B.shape[1]), np.float64)
    for k0 in range(0, A.shape[1], block):
        s = acc + A64[:, k0:k0 + block] @ B64[k0:k0 + block]    # exact here (<= 53 bits)
        acc = s.astype(np.float16).astype(np.float64)           # one RNE per instruction
    return acc

for K in (64, 256, 1024):
    for scale in (1.0, 8.0):
        A, B, _ = synth.problem(128, 256, K, "f16", seed=3)
        A = (A.astype(np.float32) * scale).astype(np.float16)
        dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
        dC = torch.zeros((128, 256), dtype=torch.float32, device="cuda")
        g.gemm_f16(dA, dB, dC, accum_f16=True, promote_k=-1, config="solo_128x256")
        torch.cuda.synchronize()
        got = dC.cpu().numpy().astype(np.float64)
        rec = {"K": K, "scale": scale}
        for blk in (16, 8, 32):
            em = emulate(A, B, blk)
            rec[f"match_block{blk}"] = float((got == em).mean())
        em = emulate(A, B, 16)
        bad = got != em
        if bad.any():
            ulp = np.abs(got[bad] - em[bad]) / np.spacing(np.abs(em[bad]).astype(np.float16)).astype(np.float64)
            rec["mismatch_ulps_max"] = float(ulp.max()); rec["mismatch_count"] = int(bad.sum())
        print(json.dumps(rec), flush=True)

def rz32(x):
    f = x.astype(np.float32)                       # RNE
    over = np.abs(f.astype(np.float64)) > np.abs(x)  # rounded away from zero -> step back
    f[over] = np.nextafter(f[over], np.float32(0))
    return f.astype(np.float64)

# the F32 accumulator (default idesc) under the same protocol: RZ or RNE per instruction?
for K in (256, 1024, 4096):
    A, B, _ = synth.problem(128, 256, K, "f32", seed=4)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    dC = torch.zeros((128, 256), dtype=torch.float32, device="cuda")
    g.gemm_f16(dA, dB, dC, promote_k=-1, config="solo_128x256")
    torch.cuda.synchronize()
    got = dC.cpu().numpy().astype(np.float64)
    A64, B64 = A.astype(np.float64), B.astype(np.float64)
    rec = {"f32_acc_K": K}
    for name, rnd in (("rz", rz32), ("rne", lambda x: x.astype(np.float32).astype(np.float64))):
        acc = np.zeros_like(got)
        for k0 in range(0, K, 16):
            acc = rnd(acc + A64[:, k0:k0 + 16] @ B64[k0:k0 + 16])
        rec[f"match_{name}_per_k16"] = float((got == acc).mean())
    print(json.dumps(rec), flush=True)

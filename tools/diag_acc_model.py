"""EXPERIMENT: fit the tensor core's per-instruction accumulation model.
Per k16 instruction and output element: terms = {acc, 16 exact products};
each term is truncated toward zero to a multiple of 2^(e_max - p + 1) (e_max: the
exponent of the largest term's leading bit), the truncated terms are summed exactly,
and the sum is rounded to the accumulator format (RZ or RNE).  Reports the bitwise
match rate of each (p, rounding) against the GPU (promote_k=-1, C_in = 0, one chain)."""
import os, sys, json
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch
import synth
import paper_2108_13191_b200 as g

def to_fmt(x, fmt, mode):
    f = x.astype(fmt)
    if mode == "rz":
        over = np.abs(f.astype(np.float64)) > np.abs(x)
        f[over] = np.nextafter(f[over], fmt(0))
    return f.astype(np.float64)

def model(A, B, p, fmt, mode, emax_from="all", acc_trunc=True, group=16):
    """group: products summed per alignment step (16 = one instruction; 8/4 = sub-steps)."""
    A64, B64 = A.astype(np.float64), B.astype(np.float64)
    acc = np.zeros((A.shape[0], B.shape[1]))
    for k0 in range(0, A.shape[1], group):
        prods = A64[:, None, k0:k0 + group] * B64[k0:k0 + group].T[None, :, :]   # exact
        terms = np.concatenate([acc[:, :, None], prods], axis=2)
        mx = np.abs(terms if emax_from == "all" else prods).max(axis=2)
        _, e = np.frexp(np.where(mx > 0, mx, 1.0))
        q = np.ldexp(1.0, (e - 1) - (p - 1))[:, :, None]
        tp = np.trunc(prods / q) * q
        s = tp.sum(axis=2) + (np.trunc(acc / q[:, :, 0]) * q[:, :, 0] if acc_trunc else acc)
        acc = to_fmt(s, fmt, mode)
    return acc

out = []
for acc_name, fmt, kw in (("f32", np.float32, {}), ("f16", np.float16, {"accum_f16": True})):
    for K in (64, 512):
        A, B, _ = synth.problem(64, 128, K, "f32", seed=6)
        dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
        dC = torch.zeros((64, 128), dtype=torch.float32, device="cuda")
        g.gemm_f16(dA, dB, dC, promote_k=-1, config="solo_128x64", **kw)
        torch.cuda.synchronize()
        got = dC.cpu().numpy().astype(np.float64)
        best = []
        for p in (24, 25, 26, 27, 28):
            for mode in ("rz", "rne"):
                for ef in ("all", "prods"):
                    for at in (True, False):
                        for grp in (16, 8, 4):
                            best.append((float((model(A, B, p, fmt, mode, ef, at, grp) == got).mean()), p, mode, ef, at, grp))
        best.sort(reverse=True)
        print(json.dumps({"acc": acc_name, "K": K, "top": best[:5]}), flush=True)

"""The paper's square sweep M=N=K=1024..16384 step 256 (fig:ampere-mixed
P:915-922, fig:ampere-half P:968-975) on B200, both modes, with cuBLAS measured in the same
process as the paper's comparison system (DIAGNOSTIC ONLY; F16: torch.addmm, the same op;
F32: torch.mm fp16->fp32 out, which skips the C_in read).  Back-to-back launches, CUDA
events, median of 3 rounds.  JSON lines on stdout."""
import os, sys, json, statistics
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch, synth
import paper_2108_13191_b200 as g

def timeit(fn, reps, rounds=3):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(rounds):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        for _ in range(reps): fn()
        e.record(); torch.cuda.synchronize()
        out.append(s.elapsed_time(e) / reps)
    return statistics.median(out)

lo, hi = int(os.environ.get("LO", "1024")), int(os.environ.get("HI", "16384"))
Abig = torch.from_numpy(synth.uniform_f16(0, 0, hi, hi)).cuda()
Bbig = torch.from_numpy(synth.uniform_f16(0, 1, hi, hi)).cuda()
for n in range(lo, hi + 1, 256):
    A = Abig[:n, :n].contiguous()
    B = Bbig[:n, :n].contiguous()
    flops = 2.0 * n ** 3
    reps = max(3, min(40, int(3e12 / flops)))
    row = {"n": n}
    for mode in ("f32", "f16"):
        C = (torch.rand(n, n, device="cuda") * 2 - 1)
        C = C if mode == "f32" else C.half()
        ms = timeit(lambda: g.gemm_f16(A, B, C), reps)
        if mode == "f32":
            cms = timeit(lambda: torch.mm(A, B, out_dtype=torch.float32), reps)
        else:
            O = torch.empty_like(C)
            cms = timeit(lambda: torch.addmm(C, A, B, out=O), reps)
        row[mode] = round(flops / ms / 1e9, 1)
        row[f"cublas_{mode}"] = round(flops / cms / 1e9, 1)
        row[f"pct_of_cublas_{mode}"] = round(100 * cms / ms, 1)
        del C
    print(json.dumps(row), flush=True)

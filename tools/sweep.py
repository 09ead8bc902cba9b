"""BASELINE.json configs[1,2,4] sweep: TFLOP/s per shape and mode (CUDA events, median of
rounds of back-to-back launches), roofline class, and -- DIAGNOSTIC ONLY, never a product
path -- cuBLAS on the same inputs in the same process.  Writes JSON lines to stdout."""
import os, sys, json, statistics
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch, synth
import paper_2108_13191_b200 as g

_mp = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "MEASURED_PEAKS.json")
_peaks = json.load(open(_mp)) if os.path.exists(_mp) else {}
PEAK_TF = float(_peaks.get("bf16_tflops", 1611.6))   # fp16 dense = bf16 rate (nominal 1:1)
HBM = float(_peaks.get("hbm_gbs", 6545.9)) * 1e9
shapes = [(1024, 1024, 1024)] + [(s, s, s) for s in range(2048, 16385, 2048)]
shapes += [(4096, 1024, 1024), (4096, 1024, 4096), (4096, 4096, 1024), (4096, 4096, 4096), (8192, 1024, 1024),
           (8192, 1024, 4096), (8192, 4096, 1024), (8192, 4096, 4096), (16384, 1024, 1024), (16384, 1024, 4096),
           (16384, 4096, 1024), (16384, 4096, 4096), (32768, 1024, 1024), (32768, 1024, 4096), (32768, 4096, 1024),
           (32768, 4096, 4096), (4097, 1024, 1024), (12345, 4096, 1024), (32767, 1024, 4096), (8192, 1000, 1000),
           (4100, 4096, 4104)]
if len(sys.argv) > 1:
    shapes = [tuple(int(x) for x in a.split("x")) for a in sys.argv[1:]]
cfg_env = os.environ.get("CONFIG", "auto")
cfg_env = int(cfg_env) if cfg_env.isdigit() else cfg_env
cublas = os.environ.get("CUBLAS", "1") == "1"

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

for (M, N, K) in shapes:
    A = torch.from_numpy(synth.uniform_f16(0, 0, M, K)).cuda()
    B = torch.from_numpy(synth.uniform_f16(0, 1, K, N)).cuda()
    flops = 2.0 * M * N * K
    reps = max(3, min(50, int(2e12 / flops)))
    for mode in ("f32", "f16"):
        C = torch.from_numpy((synth.uniform_f32 if mode == "f32" else synth.uniform_f16)(0, 2, M, N)).cuda()
        sc = 4 if mode == "f32" else 2
        byts = 2 * (M * K + K * N) + 2 * M * N * sc
        ms = timeit(lambda: g.gemm_f16(A, B, C, config=cfg_env), reps)
        tf = flops / ms / 1e9
        roof_ms = max(flops / (PEAK_TF * 1e12), byts / HBM) * 1e3
        row = {"M": M, "N": N, "K": K, "mode": mode, "config": g.pick_config(M, N, K, 0 if mode == "f32" else 1) if cfg_env == "auto" else cfg_env,
               "ms": round(ms, 5), "tflops": round(tf, 1), "bound": "tensor" if flops / byts > PEAK_TF * 1e12 / HBM else "hbm",
               "roofline_ms": round(roof_ms, 5), "frac_of_roofline": round(roof_ms / ms, 3)}
        if cublas:
            try:
                if mode == "f32":
                    cms = timeit(lambda: torch.mm(A, B, out_dtype=torch.float32), reps)
                    row["cublas_diag"] = "mm fp16->fp32 out (no C_in)"
                else:
                    O = torch.empty_like(C)
                    cms = timeit(lambda: torch.addmm(C, A, B, out=O), reps)
                    row["cublas_diag"] = "addmm f16 (C_in read)"
                row["cublas_ms"] = round(cms, 5)
                row["cublas_tflops"] = round(flops / cms / 1e9, 1)
            except Exception as ex:
                row["cublas_err"] = str(ex)[:80]
        print(json.dumps(row), flush=True)
        del C
    del A, B
    torch.cuda.empty_cache()

"""DIAGNOSTIC ONLY (never on the measured path): our kernel vs cuBLAS (torch.matmul)
in the same back-to-back protocol at n^3, with NVML clock/power samples."""
import os, sys, time, threading, statistics, json
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch, pynvml
import synth
import paper_2108_13191_b200 as g

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
steps, warm = 30, 5
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
A = torch.from_numpy(synth.uniform_f16(0, 0, n, n)).cuda()
B = torch.from_numpy(synth.uniform_f16(0, 1, n, n)).cuda()
C32 = torch.from_numpy(synth.uniform_f32(0, 2, n, n)).cuda()
C16 = C32.half()
Ab, Bb = A.bfloat16(), B.bfloat16()
O16 = torch.empty_like(C16)
flops = 2.0 * n ** 3

def sample(stop, out):
    while not stop.is_set():
        out.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
        time.sleep(0.002)

def timeit(name, fn):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    smp = []; stop = threading.Event(); t = threading.Thread(target=sample, args=(stop, smp)); t.start()
    s.record()
    for _ in range(steps): fn()
    e.record(); torch.cuda.synchronize(); stop.set(); t.join()
    ms = s.elapsed_time(e) / steps
    clk = statistics.median(x[0] for x in smp) if smp else None
    pw = max(x[1] for x in smp) if smp else None
    print(json.dumps({"name": name, "ms": round(ms, 4), "tflops": round(flops / ms / 1e9, 1), "nvml_sm_mhz_median": clk, "power_w_max": pw, "samples": len(smp)}), flush=True)
    time.sleep(1.0)

for rep in range(2):
    timeit("ours f32-acc (C f32 +=)", lambda: g.gemm_f16(A, B, C32))
    timeit("ours f16 (C f16 +=)", lambda: g.gemm_f16(A, B, C16))
    timeit("cublas fp16 matmul (out f16)", lambda: torch.matmul(A, B, out=O16))
    timeit("cublas bf16 matmul (out bf16)", lambda: torch.matmul(Ab, Bb))
    try:
        timeit("cublas addmm f16 (C f16 +=)", lambda: torch.addmm(C16, A, B, out=O16))
    except Exception as ex:
        print("addmm", ex)

"""A/B of kernel variants in the power-capped regime: each round runs every
variant back to back for ~SECS seconds while NVML samples SM clock and board
power, so the result separates per-cycle efficiency (TFLOP/s per GHz) from
the clock the variant sustains under the power cap.
VARIANTS='[{"mode":"f16","config":"pair_256x256_k128"},{"mode":"f16","config":"pair_256x512"}]' python tools/ab_power.py"""
import json
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import pynvml
import torch

import paper_2108_13191_b200 as g
import synth

variants = json.loads(os.environ["VARIANTS"])
rounds = int(os.environ.get("ROUNDS", "6"))
secs = float(os.environ.get("SECS", "0.4"))
M = int(os.environ.get("M", "8192")); N = int(os.environ.get("N", str(M))); K = int(os.environ.get("K", str(M)))
A = torch.from_numpy(synth.uniform_f16(0, 0, M, K)).cuda()
B = torch.from_numpy(synth.uniform_f16(0, 1, K, N)).cuda()
Cs = {"f32": torch.from_numpy(synth.uniform_f32(0, 2, M, N)).cuda(),
      "f16": torch.from_numpy(synth.uniform_f16(0, 2, M, N)).cuda()}

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())


_libs = {}


def _lib(path):
    # a variant {"lib": path} calls that build's gemm_f16 (default options) through ctypes
    if path not in _libs:
        import ctypes
        l = ctypes.CDLL(os.path.abspath(path))
        i64, vp, ci = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
        l.gemm_f16.restype = ci
        l.gemm_f16.argtypes = [i64, i64, i64, vp, i64, vp, i64, vp, i64, ci, vp]
        _libs[path] = l
    return _libs[path]


def run(v):
    if "lib" in v:
        C = Cs[v.get("mode", "f32")]
        st = torch.cuda.current_stream().cuda_stream
        r = _lib(v["lib"]).gemm_f16(M, N, K, A.data_ptr(), K, B.data_ptr(), N, C.data_ptr(), N,
                                    0 if v.get("mode", "f32") == "f32" else 1, st)
        assert r == 0, r
        return
    kw = {k: x for k, x in v.items() if k != "mode"}
    g.gemm_f16(A, B, Cs[v.get("mode", "f32")], **kw)


def sampled(v, n):
    samples = []
    stop = threading.Event()

    def poll():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
            time.sleep(0.002)

    t = threading.Thread(target=poll, daemon=True)
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    t.start()
    s.record()
    for _ in range(n):
        run(v)
    e.record()
    torch.cuda.synchronize()
    stop.set()
    t.join()
    ms = s.elapsed_time(e) / n
    tail = samples[len(samples) // 4:] or samples   # skip the NVML lag at the start
    return ms, statistics.median(x[0] for x in tail), statistics.median(x[1] for x in tail)


for v in variants:
    for _ in range(3):
        run(v)
torch.cuda.synchronize()
t0 = time.time()
run(variants[0])
torch.cuda.synchronize()
per_launch = max(time.time() - t0, 1e-4)
n = max(3, int(secs / per_launch))
res = {i: [] for i in range(len(variants))}
for r in range(rounds):
    order = list(range(len(variants)))
    if r % 2:
        order.reverse()
    for i in order:
        res[i].append(sampled(variants[i], n))
for i, v in enumerate(variants):
    ms = statistics.median(x[0] for x in res[i])
    mhz = statistics.median(x[1] for x in res[i])
    w = statistics.median(x[2] for x in res[i])
    tf = 2 * M * N * K / ms / 1e9
    print(json.dumps({"variant": v, "shape": [M, N, K], "launches_per_round": n, "ms_median": round(ms, 4),
                      "tflops": round(tf, 1), "sm_mhz": mhz, "watts": round(w), "tflops_per_ghz": round(tf / mhz * 1000, 1),
                      "rounds": [[round(a, 4), b, round(c)] for a, b, c in res[i]]}), flush=True)

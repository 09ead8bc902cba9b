"""A/B of library builds on bench.py's end-to-end step (gemm_f16_host from pinned host
buffers: F32 call copying A, B, C; F16 call with A, B resident), one process, one box.
LIBS='name=path,...' python tools/e2e_ab.py"""
import ctypes, os, statistics, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
n = int(os.environ.get("M", "8192"))
libs = {}
for item in os.environ["LIBS"].split(","):
    name, path = item.split("=")
    l = ctypes.CDLL(os.path.abspath(path))
    i64, vp, ci = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
    l.gemm_f16_host.restype = ci
    l.gemm_f16_host.argtypes = [i64, i64, i64, vp, i64, vp, i64, vp, i64, ci, vp, i64, vp, i64, vp, i64, vp]
    libs[name] = l
hA = torch.rand(n, n).half().pin_memory(); hB = torch.rand(n, n).half().pin_memory()
hC32 = torch.rand(n, n).pin_memory(); hC16 = torch.rand(n, n).half().pin_memory()
dA = torch.empty(n, n, dtype=torch.half, device="cuda"); dB = torch.empty_like(dA)
dC32 = torch.empty(n, n, device="cuda"); dC16 = torch.empty(n, n, dtype=torch.half, device="cuda")
st = torch.cuda.current_stream().cuda_stream
def step(l):
    r = l.gemm_f16_host(n, n, n, hA.data_ptr(), n, hB.data_ptr(), n, hC32.data_ptr(), n, 0,
                        dA.data_ptr(), n, dB.data_ptr(), n, dC32.data_ptr(), n, st)
    assert r == 0, r
    r = l.gemm_f16_host(n, n, n, None, n, None, n, hC16.data_ptr(), n, 1,
                        dA.data_ptr(), n, dB.data_ptr(), n, dC16.data_ptr(), n, st)
    assert r == 0, r
res = {k: [] for k in libs}
for k, l in libs.items():
    step(l)
torch.cuda.synchronize()
for r in range(int(os.environ.get("ROUNDS", "5"))):
    for k, l in (libs.items() if r % 2 == 0 else reversed(list(libs.items()))):
        torch.cuda.synchronize(); t = time.perf_counter()
        for _ in range(3): step(l)
        torch.cuda.synchronize(); res[k].append((time.perf_counter() - t) / 3 * 1e3)
for k, v in res.items():
    ms = statistics.median(v)
    print(f"{k}: {ms:.2f} ms per step, {2 * 2 * n ** 3 / (ms * 1e-3) / 1e12:.1f} TFLOP/s e2e, all {[round(x, 2) for x in v]}")

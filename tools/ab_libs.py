"""A/B of different builds of the library in ONE process on ONE box (box-to-box
variance is large): LIBS='name=path,...' MODES=f32,f16; round-robin blocks of
back-to-back gemm_f16 calls with default options; medians."""
import os, sys, json, ctypes, statistics
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch, synth
libs = {}
for item in os.environ["LIBS"].split(","):
    name, path = item.split("=")
    l = ctypes.CDLL(os.path.abspath(path))
    i64, vp, ci = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
    l.gemm_f16.restype = ci
    l.gemm_f16.argtypes = [i64, i64, i64, vp, i64, vp, i64, vp, i64, ci, vp]
    libs[name] = l
modes = os.environ.get("MODES", "f32,f16").split(",")
rounds = int(os.environ.get("ROUNDS", "5")); reps = int(os.environ.get("REPS", "20"))
M = int(os.environ.get("M", "8192")); N = int(os.environ.get("N", str(M))); K = int(os.environ.get("K", str(M)))
A = torch.from_numpy(synth.uniform_f16(0, 0, M, K)).cuda()
B = torch.from_numpy(synth.uniform_f16(0, 1, K, N)).cuda()
Cs = {"f32": torch.from_numpy(synth.uniform_f32(0, 2, M, N)).cuda(), "f16": torch.from_numpy(synth.uniform_f16(0, 2, M, N)).cuda()}
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
def run(l, m):
    C = Cs[m]
    r = l.gemm_f16(M, N, K, A.data_ptr(), K, B.data_ptr(), N, C.data_ptr(), N, 0 if m == "f32" else 1, st)
    assert r == 0, r
keys = [(n, m) for n in libs for m in modes]
res = {k: [] for k in keys}
for k in keys:
    for _ in range(3): run(libs[k[0]], k[1])
torch.cuda.synchronize()
for r in range(rounds):
    for k in keys:
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        for _ in range(reps): run(libs[k[0]], k[1])
        e.record(); torch.cuda.synchronize()
        res[k].append(s.elapsed_time(e) / reps)
for k in keys:
    ms = statistics.median(res[k])
    print(json.dumps({"lib": k[0], "mode": k[1], "shape": [M, N, K], "ms_median": round(ms, 4),
                      "tflops": round(2 * M * N * K / ms / 1e9, 1), "ms_all": [round(x, 4) for x in res[k]]}), flush=True)

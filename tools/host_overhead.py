"""DIAGNOSTIC: host-side cost per call of the binding layers (1024^3, F16)."""
import os, sys, time, ctypes
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch, synth
import paper_2108_13191_b200 as g
n = 1024
A = torch.from_numpy(synth.uniform_f16(0, 0, n, n)).cuda()
B = torch.from_numpy(synth.uniform_f16(0, 1, n, n)).cuda()
C = torch.from_numpy(synth.uniform_f16(0, 2, n, n)).cuda()
lib = g.load_library()
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
pa, pb, pc = A.data_ptr(), B.data_ptr(), C.data_ptr()
def bench(name, fn, reps=2000):
    for _ in range(50): fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps): fn()
    dt = (time.perf_counter() - t) / reps
    torch.cuda.synchronize()
    print(f"{name:60s} {dt*1e6:7.2f} us/call")
bench("python wrapper g.gemm_f16", lambda: g.gemm_f16(A, B, C))
bench("raw ctypes lib.gemm_f16 (precomputed args)", lambda: lib.gemm_f16(n, n, n, pa, n, pb, n, pc, n, 1, st))
bench("raw ctypes, M=0 quick return (ctypes cost only)", lambda: lib.gemm_f16(0, n, n, pa, n, pb, n, pc, n, 1, st))
bench("torch.cuda.current_stream().cuda_stream", lambda: torch.cuda.current_stream().cuda_stream)
bench("with torch.cuda.device(C.device): pass", lambda: torch.cuda.device(C.device).__enter__())

"""DIAGNOSTIC: per-tile timeline of CTA 0 (globaltimer ns) for one shape/mode."""
import os, sys, json
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch, synth
import paper_2108_13191_b200 as g
M, N, K = (int(x) for x in sys.argv[1].split("x"))
mode = sys.argv[2]
kw = json.loads(sys.argv[3]) if len(sys.argv) > 3 else {}
A = torch.from_numpy(synth.uniform_f16(0, 0, M, K)).cuda()
B = torch.from_numpy(synth.uniform_f16(0, 1, K, N)).cuda()
C = torch.from_numpy((synth.uniform_f32 if mode == "f32" else synth.uniform_f16)(0, 2, M, N)).cuda()
tr = torch.zeros(512, dtype=torch.int64, device="cuda")
CTA = int(os.environ.get("TRACE_CTA", "0"))   # CTA to trace (rank 0 of a pair: even)
tr[8 * 63 + 7] = CTA
if os.environ.get("TRACE_LIB"):   # trace another build of the library (same ABI)
    g._build.LIB = os.path.abspath(os.environ["TRACE_LIB"]); g._lib = None; g.load_library(build_if_missing=False)
for _ in range(5): g.gemm_f16(A, B, C, **kw)
g.gemm_f16(A, B, C, trace=tr, **kw)
torch.cuda.synchronize()
t = tr.cpu().numpy().reshape(64, 8)
t0 = t[0, 0]
e = t[62]
print(f"CTA{CTA}: entry {(e[0]-t0)/1000:.2f} us, setup done {(e[1]-t0)/1000:.2f}, epilogue stores drained {(e[3]-t0)/1000:.2f}, exit {(e[2]-t0)/1000:.2f}")
import time
torch.cuda.synchronize()
t_h = time.perf_counter()
for _ in range(200): g.gemm_f16(A, B, C, **kw)
t_h = (time.perf_counter() - t_h) / 200
torch.cuda.synchronize()
print(f"host enqueue time per gemm_f16 call (python + C ABI + launch): {t_h*1e6:.1f} us")
print(f"{M}x{N}x{K} {mode} {kw}: columns (us from MMA start of tile 0): mma_begin acce_ok mma_end | epi_begin accfull_last drained stored")
for i in range(62):
    if t[i, 0] == 0: break
    r = [(x - t0) / 1000 if x else float('nan') for x in t[i, :7]]
    cyc = int(t[i, 7]); ns = t[i, 2] - t[i, 0]
    kb = -(-K // 64)
    print(f"tile {i:2d}: " + " ".join(f"{x:8.2f}" for x in r[:3]) + " | " + " ".join(f"{x:8.2f}" for x in r[3:7])
          + f" | {cyc} cyc, SM clock {cyc/max(ns,1):.3f} GHz, {cyc/kb:.0f} cyc per k-block")

"""One launch (after 2 warm-ups) of a variant, for ncu / compute-sanitizer runs.
Args: JSON kwargs; extra keys M, N, K, mode, pad (leading-dim padding in elements,
makes a ragged-N edge possible), gather_peers (run gemm_f16_gather with that many
same-device peer buffers)."""
import os, sys, json
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch, synth
import paper_2108_13191_b200 as g
v = json.loads(sys.argv[1]) if len(sys.argv) > 1 else {}
M = int(v.pop("M", 8192)); N = int(v.pop("N", M)); K = int(v.pop("K", M)); mode = v.pop("mode", "f32")
pad = int(v.pop("pad", 0)); peers = int(v.pop("gather_peers", 0))
def padded(x, p):
    ld = -(-(x.shape[1] + p) // 8) * 8          # 16-byte multiple for F16 and F32
    t = torch.zeros((x.shape[0], ld), dtype=x.dtype)
    t[:, : x.shape[1]] = x
    return t.cuda()[:, : x.shape[1]]
A = padded(torch.from_numpy(synth.uniform_f16(0, 0, M, K)), pad)
B = padded(torch.from_numpy(synth.uniform_f16(0, 1, K, N)), pad)
Ch = torch.from_numpy((synth.uniform_f32 if mode == "f32" else synth.uniform_f16)(0, 2, M, N))
C = padded(Ch, pad)
if peers:
    bufs = [padded(Ch, pad) for _ in range(peers)]
    for _ in range(3): g.gemm_f16_gather(A, B, C, 0, peers=bufs)
else:
    for _ in range(3): g.gemm_f16(A, B, C, **v)
torch.cuda.synchronize()

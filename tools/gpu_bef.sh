#!/bin/bash
LIBS=bn=tools/libgemm_bn.so,bf=tools/libgemm_bf.so MODES=f32,f16 ROUNDS=10 REPS=12 timeout 600 python tools/ab_libs.py
LIBS=bn=tools/libgemm_bn.so,bf=tools/libgemm_bf.so MODES=f32,f16 M=16384 ROUNDS=4 REPS=3 timeout 600 python tools/ab_libs.py
for lib in bn bf; do
cat > /tmp/one_$lib.py <<PY
import ctypes, torch, sys
sys.path.insert(0, "."); import synth
l = ctypes.CDLL("tools/libgemm_$lib.so")
i64, vp, ci = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
l.gemm_f16.argtypes = [i64, i64, i64, vp, i64, vp, i64, vp, i64, ci, vp]
M = 8192
A = torch.from_numpy(synth.uniform_f16(0, 0, M, M)).cuda(); B = torch.from_numpy(synth.uniform_f16(0, 1, M, M)).cuda()
for mode, C in ((0, torch.from_numpy(synth.uniform_f32(0, 2, M, M)).cuda()), (1, torch.from_numpy(synth.uniform_f16(0, 2, M, M)).cuda())):
    for _ in range(3): l.gemm_f16(M, M, M, A.data_ptr(), M, B.data_ptr(), M, C.data_ptr(), M, mode, None)
torch.cuda.synchronize()
PY
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm -s 2 -c 4 python /tmp/one_$lib.py 2>/dev/null | grep -E "gemm_f16_sm100|dram__bytes|duration" | sed "s/^/$lib /"
done

"""CPU oracle for C += A.B with F16 inputs -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline``
leg and ``--impl reference``) may import this package.  The product package
``paper_2108_13191_b200`` never imports it and shares no code with it.

The arithmetic lives in ``oracle.c`` (plain C, IEEE double, OpenMP over rows);
this module only builds it with gcc and marshals numpy arrays.  See the header
of ``oracle.c`` for the PAPER.md passages followed (P:908-909 problem
statement, P:412-438 naive loop nest, P:926-930 / P:976-980 precisions).

``oracle_f16_to_f64`` / ``oracle_f64_to_f16_rne`` are the oracle's own binary16
decoder / encoder; they are pinned against numpy in tests/test_oracle_pins.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

ACC_F32 = 0
ACC_F16 = 1


def build(force: bool = False) -> str:
    """Compile oracle.c -> oracle/liboracle.so with gcc + OpenMP (no FMA contraction)."""
    if (not force and os.path.exists(_LIB_PATH)
            and os.path.getmtime(_LIB_PATH) >= os.path.getmtime(_SRC)):
        return _LIB_PATH
    tmp = _LIB_PATH + f".tmp{os.getpid()}"
    cmd = ["gcc", "-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
           "-fno-fast-math", "-std=c11", _SRC, "-o", tmp, "-lm"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        lib.oracle_f16_to_f64.restype = ctypes.c_double
        lib.oracle_f16_to_f64.argtypes = [ctypes.c_uint16]
        lib.oracle_f64_to_f16_rne.restype = ctypes.c_uint16
        lib.oracle_f64_to_f16_rne.argtypes = [ctypes.c_double]
        lib.oracle_bf16_to_f64.restype = ctypes.c_double
        lib.oracle_bf16_to_f64.argtypes = [ctypes.c_uint16]
        lib.oracle_num_threads.restype = ctypes.c_int
        lib.oracle_num_threads.argtypes = []
        i64 = ctypes.c_int64
        vp = ctypes.c_void_p
        lib.oracle_gemm_f16.restype = ctypes.c_int
        lib.oracle_gemm_f16.argtypes = [i64, i64, i64, vp, i64, vp, i64, vp, i64,
                                        ctypes.c_int, vp, i64, vp, vp]
        ci = ctypes.c_int
        lib.oracle_gemm_ex.restype = ci
        lib.oracle_gemm_ex.argtypes = [i64, i64, i64, vp, i64, vp, i64, vp, i64,
                                       ci, ci, ci, vp, ci, vp, i64, vp, vp]
        _lib = lib
    return _lib


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def f16_to_f64(bits: int) -> float:
    return float(_load().oracle_f16_to_f64(int(bits) & 0xFFFF))


def f64_to_f16_bits(x: float) -> int:
    return int(_load().oracle_f64_to_f16_rne(float(x)))


def bf16_to_f64(bits: int) -> float:
    return float(_load().oracle_bf16_to_f64(int(bits) & 0xFFFF))


def _as_bits16(a: np.ndarray) -> np.ndarray:
    if a.dtype == np.float16:
        return a.view(np.uint16)
    if a.dtype == np.uint16:
        return a
    raise TypeError(f"expected float16/uint16 array, got {a.dtype}")


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def gemm(A: np.ndarray, B: np.ndarray, C_in: np.ndarray, acc: int | None = None,
         rows=None, in_type: int = 0, beta: int = 1, bias=None, relu: bool = False):
    """Oracle C_out = epi(beta * C_in + A.B + bias) (NEXT #4 extensions).

    A: (M, K) float16 (or uint16 bfloat16 bits with in_type=1; row stride may
    exceed K), B: (K, N) likewise, C_in: (M, N) float32 (F32 mode) or float16
    (F16 mode).  rows: optional row indices (default all).  beta: 1 or 0 (C_in
    ignored).  bias: optional (N,) float32.  relu: apply max(x, 0) (NaN kept).
    Returns (C_exact float64 (nrows, N), C_round (nrows, N) in C_in's dtype).
    """
    lib = _load()
    if acc is None:
        acc = ACC_F32 if C_in.dtype == np.float32 else ACC_F16
    want = np.float32 if acc == ACC_F32 else np.float16
    if C_in.dtype != want:
        raise TypeError(f"C_in dtype {C_in.dtype} does not match acc mode {acc}")
    M, K = A.shape
    K2, N = B.shape
    if K2 != K or C_in.shape != (M, N):
        raise ValueError("shape mismatch")
    for name, t in (("A", A), ("B", B), ("C_in", C_in)):
        if t.ndim != 2 or (t.size > 0 and t.shape[1] > 1 and t.strides[1] != t.itemsize):
            raise ValueError(f"{name} must be row-major with unit column stride")
    Ab, Bb = _as_bits16(A), _as_bits16(B)
    lda = A.strides[0] // 2 if (M > 1 and A.size) else max(K, 1)
    ldb = B.strides[0] // 2 if (K > 1 and B.size) else max(N, 1)
    ldc = C_in.strides[0] // C_in.itemsize if (M > 1 and C_in.size) else max(N, 1)
    if A.size == 0:
        Ab = np.zeros(1, np.uint16)
    if B.size == 0:
        Bb = np.zeros(1, np.uint16)
    if rows is None:
        rows_arr = None
        nrows = M
    else:
        rows_arr = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
        nrows = rows_arr.shape[0]
    bias_arr = None if bias is None else np.ascontiguousarray(np.asarray(bias, dtype=np.float32))
    if bias_arr is not None and bias_arr.shape != (N,):
        raise ValueError("bias must have N elements")
    C_exact = np.empty((nrows, N), dtype=np.float64)
    C_round = np.empty((nrows, N), dtype=want)
    st = lib.oracle_gemm_ex(M, N, K, _ptr(Ab), lda, _ptr(Bb), ldb, _ptr(C_in), ldc,
                            int(acc), int(in_type), int(beta),
                            None if bias_arr is None else _ptr(bias_arr), int(bool(relu)),
                            None if rows_arr is None else _ptr(rows_arr),
                            nrows, _ptr(C_exact), _ptr(C_round))
    if st != 0:
        raise ValueError(f"oracle_gemm_ex rejected its arguments (status {st})")
    return C_exact, C_round


def timed_gemm(A, B, C_in, acc=None, rows=None):
    """gemm() plus host wall-clock seconds and the thread count used."""
    t0 = time.perf_counter()
    out = gemm(A, B, C_in, acc, rows)
    return out, time.perf_counter() - t0, num_threads()

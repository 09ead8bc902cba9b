"""B200-native (sm_100a) tensor-core GEMM: C += A.B with F16 inputs, F32 or F16 C.

The one hot path of arXiv 2108.13191 (Sec. 4: "C = AB + C,
all three matrices ... row-major"; F32 accumulate P:926-930, F16 P:976-980),
re-designed for Blackwell: a persistent, warp-specialised kernel (TMA producer,
single-thread tcgen05.mma issuer with TMEM accumulators, epilogue warpgroup)
behind the C ABI declared in include/gemm_f16.h.

This module is argument marshalling only: torch supplies device memory and
streams; every arithmetic step runs in libgemm_f16.so.  If the library is
missing the import of the binding fails loudly -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

from . import _build

__all__ = ["gemm_f16", "gemm_f16_gather", "gemm_f16_host", "GemmError", "ACC_F32", "ACC_F16", "CONFIGS",
           "config_info", "pick_config", "library_path", "load_library", "last_launches"]

ACC_F32 = 0
ACC_F16 = 1
CONFIGS = {
    "auto": 0,
    "pair_256x256": 1,
    "pair_256x128": 2,
    "solo_128x256": 3,
    "solo_128x128": 4,
    "solo_128x64": 5,
    "pair_256x256_s5": 6,
    "pair_256x256_s4": 7,
    "pair_256x256_k128": 8,
    "pair_256x512": 9,   # AUTO picks it for F16 C; F32 C is selectable (measured slower)
    "splitk_128x256_s2": 10,
    "splitk_128x256_s4": 11,
    "splitk_128x128_s4": 12,
    "solo_128x64_mc4": 13,
    "solo_128x128_mc4": 14,
    "splitk_128x128_s2": 15,
    "pair2_256x256_mcb": 16,   # B multicast across two CTA pairs (4-CTA clusters); not picked
    "pair2_256x256_mch": 17,   # the same kernel, preferred 4-CTA / regular 2-CTA clusters (all SMs)
}
_STATUS = {0: "GEMM_OK", 1: "GEMM_ERR_INVALID_VALUE", 2: "GEMM_ERR_MISALIGNED",
           3: "GEMM_ERR_UNSUPPORTED_DEVICE", 4: "GEMM_ERR_CUDA"}

EXPORTED_SYMBOLS = ("gemm_f16", "gemm_f16_ex", "gemm_f16_gather", "gemm_f16_host", "gemm_f16_pick_config",
                    "gemm_f16_pick_config_for",
                    "gemm_f16_config_info", "gemm_f16_last_launches", "gemm_status_string",
                    "gemm_last_cuda_error")
# include/gemm_f16_diag.h (diagnostic entry points; never change a result)
DIAG_SYMBOLS = ("gemm_f16_diag_set_trace", "gemm_f16_diag_sk_window_base", "gemm_f16_diag_sk_window_slots",
                "gemm_f16_diag_sk_pool_slots")


class GemmError(RuntimeError):
    def __init__(self, status: int, cuda_error: int = 0):
        self.status = status
        self.cuda_error = cuda_error
        msg = _STATUS.get(status, f"status {status}")
        if status == 4:
            msg += f" (cudaError {cuda_error})"
        super().__init__(msg)


class _Options(ctypes.Structure):
    """gemm_options_t (include/gemm_f16.h), field for field."""
    _fields_ = [("config", ctypes.c_int), ("max_clusters", ctypes.c_int), ("group_m", ctypes.c_int),
                ("promote_k", ctypes.c_int), ("in_type", ctypes.c_int), ("beta0", ctypes.c_int),
                ("relu", ctypes.c_int), ("bias", ctypes.c_void_p), ("accum_f16", ctypes.c_int),
                ("stream_k", ctypes.c_int), ("ring_stages", ctypes.c_int), ("acc_bufs", ctypes.c_int),
                ("l2_hints", ctypes.c_int), ("pdl", ctypes.c_int), ("raster", ctypes.c_int),
                ("c_reduce", ctypes.c_int), ("tail_ring", ctypes.c_int), ("swizzle", ctypes.c_int),
                ("warp_specialize", ctypes.c_int)]


# the option keywords of gemm_f16 that map 1:1 onto gemm_options_t ints (0 = default)
_INT_OPTS = ("max_clusters", "group_m", "promote_k", "stream_k", "ring_stages", "acc_bufs", "l2_hints", "pdl",
             "raster", "c_reduce", "tail_ring", "swizzle", "warp_specialize")


_lib = None


def library_path() -> str:
    return _build.LIB


def load_library(build_if_missing: bool = True):
    """Load libgemm_f16.so (building it with nvcc if stale).  Raises if unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    if build_if_missing:
        try:
            _build.build()
        except (OSError, RuntimeError) as e:  # nvcc missing on a box with a prebuilt .so
            if not os.path.exists(_build.LIB):
                raise RuntimeError(f"libgemm_f16.so is missing and cannot be built: {e}") from e
    if not os.path.exists(_build.LIB):
        raise RuntimeError(f"libgemm_f16.so not found at {_build.LIB}; run __graft_entry__.build()")
    lib = ctypes.CDLL(_build.LIB)
    i64, vp, ci = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
    lib.gemm_f16.restype = ci
    lib.gemm_f16.argtypes = [i64, i64, i64, vp, i64, vp, i64, vp, i64, ci, vp]
    lib.gemm_f16_ex.restype = ci
    lib.gemm_f16_ex.argtypes = [i64, i64, i64, vp, i64, vp, i64, vp, i64, ci, vp, ctypes.POINTER(_Options)]
    lib.gemm_f16_gather.restype = ci
    lib.gemm_f16_gather.argtypes = [i64, i64, i64, vp, i64, vp, i64, i64, i64, vp, i64, ctypes.POINTER(vp), ci, ci, vp]
    lib.gemm_f16_host.restype = ci
    lib.gemm_f16_host.argtypes = [i64, i64, i64, vp, i64, vp, i64, vp, i64, ci, vp, i64, vp, i64, vp, i64, vp]
    lib.gemm_f16_pick_config.restype = ci
    lib.gemm_f16_pick_config.argtypes = [i64, i64, i64, ci]
    lib.gemm_f16_pick_config_for.restype = ci
    lib.gemm_f16_pick_config_for.argtypes = [i64, i64, i64, ci, ci]
    lib.gemm_f16_config_info.restype = ci
    lib.gemm_f16_config_info.argtypes = [ci, ci] + [ctypes.POINTER(ci)] * 5
    lib.gemm_f16_last_launches.restype = ci
    lib.gemm_f16_last_launches.argtypes = []
    lib.gemm_status_string.restype = ctypes.c_char_p
    lib.gemm_status_string.argtypes = [ci]
    lib.gemm_last_cuda_error.restype = ci
    lib.gemm_last_cuda_error.argtypes = []
    lib.gemm_f16_diag_set_trace.restype = ci
    lib.gemm_f16_diag_set_trace.argtypes = [vp]
    u32 = ctypes.c_uint32
    lib.gemm_f16_diag_sk_window_base.restype = u32
    lib.gemm_f16_diag_sk_window_base.argtypes = [u32]
    lib.gemm_f16_diag_sk_window_slots.restype = u32
    lib.gemm_f16_diag_sk_window_slots.argtypes = []
    lib.gemm_f16_diag_sk_pool_slots.restype = u32
    lib.gemm_f16_diag_sk_pool_slots.argtypes = []
    _lib = lib
    return lib


def _check(status: int):
    if status != 0:
        raise GemmError(status, _lib.gemm_last_cuda_error() if status == 4 else 0)


def _ld(t, name):
    """Leading dimension (elements) of a row-major 2-D tensor with unit column stride."""
    if t.dim() != 2:
        raise ValueError(f"{name} must be 2-D")
    if t.size(1) > 1 and t.stride(1) != 1:
        raise ValueError(f"{name} must be row-major (unit column stride)")
    if t.size(0) > 1:
        return t.stride(0)
    # a single row: the stride is never used to address memory, but TMA still
    # needs a 16-byte multiple >= the row length
    per16 = 16 // t.element_size()
    return -(-max(t.size(1), 1) // per16) * per16


def _stream_handle(stream, device_index):
    import torch
    if stream is None:
        return torch._C._cuda_getCurrentRawStream(device_index)
    return stream.cuda_stream


def _acc_of(C):
    import torch
    if C.dtype == torch.float32:
        return ACC_F32
    if C.dtype == torch.float16:
        return ACC_F16
    raise TypeError(f"C must be float32 (F32 accumulate) or float16 (F16), got {C.dtype}")


def _check_operands(A, B, C, names=("A", "B", "C")):
    """Device, dtype and placement checks shared by every entry point (no CPU fallback)."""
    import torch
    for name, t in zip(names, (A, B, C)):
        if not t.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if A.dtype not in (torch.float16, torch.bfloat16) or B.dtype != A.dtype:
        raise TypeError(f"{names[0]} and {names[1]} must both be torch.float16 or both torch.bfloat16")
    if A.device != C.device or B.device != C.device:
        raise ValueError(f"{', '.join(names)} must be on the same CUDA device")
    return _acc_of(C)


_fast_types = None   # (torch.float16, torch.float32, _cuda_getDevice, _cuda_getCurrentRawStream), set on first use
_fastbind = None     # csrc/fastbind.cpp, when built (_build.build_fastbind); else the ctypes path below
_fastbind_tried = False


def _load_fastbind():
    """Import the in-tree torch extension of the default call, if it was built, and hand it the
    library's gemm_f16 entry point.  Absent or unloadable: None (the ctypes path is used)."""
    global _fastbind, _fastbind_tried
    _fastbind_tried = True
    if _lib is None or not os.path.exists(_build.FASTBIND_SO):
        return None
    try:
        import importlib.util
        import torch  # noqa: F401  (the extension resolves libtorch symbols)
        spec = importlib.util.spec_from_file_location("gemm_f16_fastbind", _build.FASTBIND_SO)
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        mod.set_entry(ctypes.cast(_lib.gemm_f16, ctypes.c_void_p).value)
        mod.set_entry_ex(ctypes.cast(_lib.gemm_f16_ex, ctypes.c_void_p).value)
        _fastbind = mod
    except Exception:   # a stale or foreign build: keep the ctypes path
        _fastbind = None
    return _fastbind


def _gemm_f16_fast(A, B, C):
    """The default call (C += A @ B, F16 inputs, torch's current stream, no options) with the
    fewest tensor queries: returns C, or None when any check needs the general path (which
    then raises the precise error).  The arguments and checks are the general path's."""
    global _fast_types
    lib = _lib
    if lib is None:
        return None
    if _fast_types is None:
        import torch
        _fast_types = (torch.float16, torch.float32, torch._C._cuda_getDevice, torch._C._cuda_getCurrentRawStream)
    f16, f32, get_device, raw_stream = _fast_types
    if A.dtype is not f16 or B.dtype is not f16:
        return None
    cdt = C.dtype
    acc = ACC_F32 if cdt is f32 else ACC_F16 if cdt is f16 else None
    if acc is None:
        return None
    dev = C.get_device()   # (-1 for a CPU tensor)
    if dev < 0 or A.get_device() != dev or B.get_device() != dev or dev != get_device():
        return None
    if A.dim() != 2 or B.dim() != 2 or C.dim() != 2:
        return None
    M, K = A.shape
    K2, N = B.shape
    if K2 != K or C.shape[0] != M or C.shape[1] != N or M < 2 or N < 2 or K < 2:
        return None
    sa, sb, sc = A.stride(), B.stride(), C.stride()
    if sa[1] != 1 or sb[1] != 1 or sc[1] != 1:
        return None
    st = lib.gemm_f16(M, N, K, A.data_ptr(), sa[0], B.data_ptr(), sb[0], C.data_ptr(), sc[0], acc, raw_stream(dev))
    if st:
        _check(st)
    return C


def gemm_f16(A, B, C, stream=None, config=0, beta: int = 1, bias=None, relu: bool = False,
             accum_f16: bool = False, trace=None, **opts):
    """In place: C += A @ B on the GPU (enqueued on `stream`, default: torch's current).

    A: (M, K) torch.float16 or torch.bfloat16 CUDA, B: (K, N) of the same dtype,
    C: (M, N) float32 or float16 CUDA; all row-major with unit column stride (row
    strides = leading dims).  Fused epilogue: C <- relu?(beta * C + A @ B + bias),
    beta in {1, 0}, bias an (N,) float32 CUDA tensor.  config: a name in CONFIGS or
    its id (0 = auto).  accum_f16 (EXPERIMENT): the tensor core accumulates in
    binary16 (DESIGN R16).  Further keyword options (each 0 = default): the ints of
    gemm_options_t named in _INT_OPTS (max_clusters, group_m, promote_k, stream_k and
    the ablation knobs).  trace (DIAGNOSTIC): a CUDA int64 tensor of 512 elements that
    receives per-tile timestamps (include/gemm_f16_diag.h).  Raises GemmError on a
    non-zero status.
    """
    if stream is None and not opts and not accum_f16 and trace is None and beta in (0, 1):
        # the extension (csrc/fastbind.cpp) takes the default call and the common options (a
        # configuration, beta = 0, ReLU, a bias); it declines (-1) anything else, which then
        # takes the general path below and gets its precise error there
        fb = _fastbind if _fastbind_tried else (_load_fastbind() if _lib is not None else None)
        plain = config == 0 and beta == 1 and bias is None and not relu
        if fb is not None:
            if plain:
                st = fb.gemm_default(A, B, C)
            else:
                cfg = CONFIGS[config] if isinstance(config, str) else int(config)
                st = fb.gemm_options(A, B, C, cfg, 1 - int(beta), int(bool(relu)), bias)
            if st == 0:
                return C
            if st > 0:
                _check(st)
        elif plain and _gemm_f16_fast(A, B, C) is not None:
            return C
    import torch
    lib = load_library()
    bad = set(opts) - set(_INT_OPTS)
    if bad:
        raise TypeError(f"unknown options {sorted(bad)}")
    acc = _check_operands(A, B, C)
    in_type = 1 if A.dtype == torch.bfloat16 else 0
    if beta not in (0, 1):
        raise ValueError("beta must be 1 (C += A.B) or 0 (C = A.B)")
    if bias is not None and (bias.dtype != torch.float32 or bias.dim() != 1 or bias.numel() != B.shape[1]
                             or not bias.is_cuda or bias.stride(0) != 1 or bias.device != C.device):
        raise ValueError("bias must be a contiguous float32 CUDA vector of N elements on C's device")
    M, K = A.shape
    K2, N = B.shape
    if K2 != K or tuple(C.shape) != (M, N):
        raise ValueError(f"shape mismatch: A{tuple(A.shape)} B{tuple(B.shape)} C{tuple(C.shape)}")
    cfg = CONFIGS[config] if isinstance(config, str) else int(config)
    dev = C.device.index
    cur = torch._C._cuda_getDevice()
    ctx = torch.cuda.device(dev) if dev != cur else None
    if ctx is not None:
        ctx.__enter__()
    try:
        sh = _stream_handle(stream, dev)
        if trace is not None:
            if not (trace.is_cuda and trace.dtype == torch.int64 and trace.numel() >= 512):
                raise ValueError("trace must be a CUDA int64 tensor of >= 512 elements")
            lib.gemm_f16_diag_set_trace(trace.data_ptr())
        if (cfg == 0 and in_type == 0 and beta == 1 and bias is None and not relu and not accum_f16
                and not any(opts.values())):
            st = lib.gemm_f16(M, N, K, A.data_ptr(), _ld(A, "A"), B.data_ptr(), _ld(B, "B"),
                              C.data_ptr(), _ld(C, "C"), acc, sh)
        else:
            o = _Options(config=cfg, in_type=in_type, beta0=1 - int(beta), relu=int(bool(relu)),
                         bias=None if bias is None else ctypes.c_void_p(bias.data_ptr()),
                         accum_f16=int(bool(accum_f16)), **{k: int(v) for k, v in opts.items()})
            st = lib.gemm_f16_ex(M, N, K, A.data_ptr(), _ld(A, "A"), B.data_ptr(), _ld(B, "B"),
                                 C.data_ptr(), _ld(C, "C"), acc, sh, ctypes.byref(o))
        if trace is not None:
            lib.gemm_f16_diag_set_trace(None)   # (disarm if the call failed before launching)
    finally:
        if ctx is not None:
            ctx.__exit__(None, None, None)
    _check(st)
    return C


def gemm_f16_gather(A, B_r, C, n0: int, peers=(), stream=None):
    """This rank's share of an N-sharded C += A.B fused with the all-gather of C.

    C: this rank's full (M, N) buffer (float32 or float16, CUDA); the rank owns
    columns [n0, n0 + B_r.shape[1]).  C[:, n0:n0+nr] += A @ B_r, and each finished
    tile is also stored into every peer buffer at the same columns.  `peers`:
    device addresses (ints) or tensors of the other ranks' full C buffers, same
    shape / dtype / row stride, mapped into this process (e.g. torch symmetric
    memory `buffer_ptrs`) or other buffers on this device.  At most 7.
    """
    import torch
    lib = load_library()
    acc = _check_operands(A, B_r, C, names=("A", "B_r", "C"))
    if A.dtype != torch.float16:
        raise TypeError("gemm_f16_gather takes binary16 A and B_r")
    M, K = A.shape
    K2, nr = B_r.shape
    if K2 != K or C.shape[0] != M or n0 < 0 or n0 + nr > C.shape[1]:
        raise ValueError("shape mismatch")
    ptrs = [int(x.data_ptr()) if hasattr(x, "data_ptr") else int(x) for x in peers]
    arr = (ctypes.c_void_p * max(1, len(ptrs)))(*ptrs)
    dev = C.device.index
    ctx = torch.cuda.device(dev) if dev != torch._C._cuda_getDevice() else None
    if ctx is not None:
        ctx.__enter__()
    try:
        st = lib.gemm_f16_gather(M, C.shape[1], K, A.data_ptr(), _ld(A, "A"), B_r.data_ptr(), _ld(B_r, "B_r"),
                                 int(n0), int(nr), C.data_ptr(), _ld(C, "C"),
                                 ctypes.cast(arr, ctypes.POINTER(ctypes.c_void_p)), len(ptrs), acc,
                                 _stream_handle(stream, dev))
    finally:
        if ctx is not None:
            ctx.__exit__(None, None, None)
    _check(st)
    return C


def gemm_f16_host(hA, hB, hC, dA, dB, dC, stream=None):
    """End-to-end path: host (pinned) A, B, C -> device scratch -> GEMM -> C back to host.

    hA/hB/hC are CPU torch tensors (float16 / float16 / float32|float16); dA/dB/dC
    are CUDA scratch tensors of the same shapes and dtypes.  hA or hB may be None:
    that operand is already resident in dA / dB (e.g. a second GEMM on the same
    operands).  Enqueued on `stream`; the caller synchronises before reading hC.
    """
    import torch
    lib = load_library()
    acc = _check_operands(dA, dB, dC, names=("dA", "dB", "dC"))
    if dA.dtype != torch.float16:
        raise TypeError("gemm_f16_host takes binary16 A and B")
    if hC.dtype != dC.dtype or hC.is_cuda:
        raise TypeError("hC must be a host tensor of dC's dtype")
    for name, h, d in (("hA", hA, dA), ("hB", hB, dB)):
        if h is not None and (h.is_cuda or h.dtype != d.dtype):
            raise TypeError(f"{name} must be a host tensor of the device scratch's dtype")
    M, K = dA.shape
    _, N = dB.shape
    if tuple(hC.shape) != (M, N) or tuple(dC.shape) != (M, N) or dB.shape[0] != K:
        raise ValueError("hC/dC must be (M, N) and dB (K, N) for dA (M, K)")
    pA = 0 if hA is None else hA.data_ptr()
    pB = 0 if hB is None else hB.data_ptr()
    lA = 0 if hA is None else _ld(hA, "hA")
    lB = 0 if hB is None else _ld(hB, "hB")
    if hA is not None and tuple(hA.shape) != (M, K) or hB is not None and tuple(hB.shape) != (K, N):
        raise ValueError("host and device operand shapes differ")
    with torch.cuda.device(dC.device):
        st = lib.gemm_f16_host(M, N, K, pA, lA, pB, lB,
                               hC.data_ptr(), _ld(hC, "hC"), acc,
                               dA.data_ptr(), _ld(dA, "dA"), dB.data_ptr(), _ld(dB, "dB"),
                               dC.data_ptr(), _ld(dC, "dC"), _stream_handle(stream, dC.device.index))
    _check(st)
    return hC


def pick_config(M: int, N: int, K: int, acc: int = ACC_F32, sm_count: int = 0) -> int:
    """Configuration gemm_f16 would use; with sm_count > 0, the table for that SM count
    evaluated on the host only (no device needed)."""
    lib = load_library()
    if sm_count > 0:
        return int(lib.gemm_f16_pick_config_for(M, N, K, acc, sm_count))
    return int(lib.gemm_f16_pick_config(M, N, K, acc))


def config_info(config, acc: int = ACC_F32) -> dict:
    lib = load_library()
    cfg = CONFIGS[config] if isinstance(config, str) else int(config)
    vals = [ctypes.c_int() for _ in range(5)]
    _check(lib.gemm_f16_config_info(cfg, acc, *[ctypes.byref(v) for v in vals]))
    keys = ("tile_m", "tile_n", "cta_group", "stages", "smem_bytes")
    return {k: v.value for k, v in zip(keys, vals)}


def last_launches() -> int:
    return int(load_library().gemm_f16_last_launches())

"""Shared helpers for the parity tests: seeded problems on the device, guard-banded
buffers, and the tolerance checks stated in BASELINE.json's north_star.

Tolerances (BASELINE.json north_star):
  F32 accumulate: max|err| <= 1e-3 * sqrt(K) * max|A| * max|B| elementwise, AND
                  ||C_gpu - C_exact||_F / ||C_exact||_F <= 1e-5
  F16 accumulate: ||C_gpu - C_exact||_F / ||C_exact||_F <= 2e-3 (worst element reported),
                  AND element by element (a Frobenius bar alone lets a whole
                  tile that lost its C_in pass at 8192^3):
                      |C_gpu - C_exact| <= 2 ulp16(|C_exact|) + delta32,
                      delta32 = (ceil(K/16) + 4) * 2^-23 * S,  S = sum_k |A_ik B_kj| + |C_in|
                  -- two binary16 ulps for the one RNE rounding to C's type (DESIGN R3),
                  plus the F32 accumulation allowance: the tensor core's accumulator
                  truncates once per K=16 step (DESIGN R4), each time by less than one
                  F32 ulp of a partial sum, and every partial sum is bounded by S; four
                  more ulps cover the promotion adds and the C_in add.
C_exact is the oracle's double-precision result over the same F16-rounded inputs.
"""
from __future__ import annotations

import numpy as np

import oracle
import synth

F32_ELEM = 1e-3
F32_FRO = 1e-5
F16_FRO = 2e-3

CANARY_F32 = np.uint32(0x7FBADBAD)   # a NaN payload no arithmetic produces
CANARY_F16 = np.uint16(0x7E5B)


def round_up(x, m):
    return -(-x // m) * m


def stats(C_gpu: np.ndarray, C_exact: np.ndarray):
    err = C_gpu.astype(np.float64) - C_exact
    den = np.linalg.norm(C_exact)
    rel = np.linalg.norm(err) / den if den > 0 else np.linalg.norm(err)
    idx = np.unravel_index(int(np.argmax(np.abs(err))), err.shape) if err.size else (0, 0)
    return {"rel_fro": float(rel), "max_abs": float(np.abs(err).max()) if err.size else 0.0,
            "worst": tuple(int(i) for i in idx), "mean_err": float(err.mean()) if err.size else 0.0}


def ulp16(x):
    """Spacing of binary16 at |x| (subnormal spacing 2^-24 below 2^-14)."""
    ax = np.abs(np.asarray(x, np.float64))
    e = np.floor(np.log2(np.maximum(ax, 2.0 ** -14)))
    return np.exp2(e - 10)


def f16_element_bound(C_exact, A, B, K: int, C_in=None, extra_roundings: int = 0):
    """Per-element F16-mode bound (module docstring).  extra_roundings: binary16
    roundings of partial sums (e.g. the R18 stream-K hand-over), each <= ulp16(S)/2."""
    Aa = np.abs(np.asarray(A, np.float32))
    Ba = np.abs(np.asarray(B, np.float32))
    S = (Aa @ Ba).astype(np.float64) * 1.01
    if C_in is not None:
        S += np.abs(np.asarray(C_in, np.float64))
    delta32 = (-(-K // 16) + 4) * 2.0 ** -23 * S
    return 2.0 * ulp16(C_exact) + delta32 + 0.5 * extra_roundings * ulp16(S)


def check(C_gpu, C_exact, A, B, acc: str, K: int, what: str = "", C_in=None, extra_roundings: int = 0):
    s = stats(C_gpu, C_exact)
    assert np.all(np.isfinite(C_gpu)), f"{what}: non-finite output"
    if acc == "f32":
        maxA = float(np.abs(A.astype(np.float32)).max()) if A.size else 0.0
        maxB = float(np.abs(B.astype(np.float32)).max()) if B.size else 0.0
        bound = F32_ELEM * np.sqrt(max(K, 1)) * maxA * maxB
        assert s["max_abs"] <= bound, f"{what}: max|err| {s['max_abs']:.3e} > {bound:.3e} ({s})"
        assert s["rel_fro"] <= F32_FRO, f"{what}: rel Frobenius {s['rel_fro']:.3e} > 1e-5 ({s})"
    else:
        assert s["rel_fro"] <= F16_FRO, f"{what}: rel Frobenius {s['rel_fro']:.3e} > 2e-3 ({s})"
        if C_gpu.size:
            err = np.abs(C_gpu.astype(np.float64) - C_exact)
            bound = f16_element_bound(C_exact, A, B, K, C_in, extra_roundings)
            bad = err > bound
            if bad.any():
                i = np.unravel_index(int(np.argmax(err - bound)), err.shape)
                raise AssertionError(f"{what}: {int(bad.sum())} elements beyond the F16 element bound; worst "
                                     f"{tuple(int(x) for x in i)}: |err| {err[i]:.4g} > {bound[i]:.4g} "
                                     f"(C_exact {C_exact[i]:.6g}, got {float(C_gpu[i]):.6g})")
            s["elem_slack_min"] = float((bound - err).min())
    return s


class Guarded:
    """A row-major (rows x cols) device matrix embedded in a larger allocation whose
    padding columns and trailing rows hold a canary bit pattern."""

    def __init__(self, host: np.ndarray, ld: int, extra_rows: int = 3):
        import torch
        self.rows, self.cols = host.shape
        self.ld = ld
        self.dtype = host.dtype
        item = host.dtype.itemsize
        if item == 4:
            canary = np.full((self.rows + extra_rows, ld), CANARY_F32, dtype=np.uint32).view(np.float32)
        else:
            canary = np.full((self.rows + extra_rows, ld), CANARY_F16, dtype=np.uint16).view(np.float16)
        canary[: self.rows, : self.cols] = host
        self.full_host = canary
        self.full = torch.from_numpy(canary.copy()).cuda()
        self.view = self.full[: self.rows, : self.cols]

    def result(self) -> np.ndarray:
        self.last = self.full.cpu().numpy()
        return self.last[: self.rows, : self.cols]

    def guard_intact(self) -> bool:
        now = self.full.cpu().numpy()
        mask = np.ones(now.shape, dtype=bool)
        mask[: self.rows, : self.cols] = False
        a = now.view(np.uint32 if now.dtype.itemsize == 4 else np.uint16)
        b = self.full_host.view(a.dtype)
        return bool(np.array_equal(a[mask], b[mask]))


def device_problem(M, N, K, acc, seed=0, pad=(0, 0, 0), extra_rows=3):
    """Seeded inputs on the device in guard-banded buffers; returns (A,B,C host, gA,gB,gC)."""
    A, B, C = synth.problem(M, N, K, acc, seed=seed)
    csz = 4 if acc == "f32" else 2
    lda = round_up(max(K, 1), 8) + pad[0]
    ldb = round_up(max(N, 1), 8) + pad[1]
    ldc = round_up(max(N, 1), 16 // csz) + pad[2]
    return A, B, C, Guarded(A, lda, extra_rows), Guarded(B, ldb, extra_rows), Guarded(C, ldc, extra_rows)


def oracle_full(A, B, C):
    return oracle.gemm(A, B, C)

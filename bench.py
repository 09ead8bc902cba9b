#!/usr/bin/env python
"""bench.py -- throughput of the hot path on B200: C += A.B, F16 inputs, at M=N=K=8192.

One step = one F32-accumulate GEMM and one F16-accumulate GEMM (both modes the
paper evaluates, Sec. 4.1 P:924-949 and Sec. 4.2; BASELINE.json
metric "GEMM TFLOP/s & % of B200 dense FP16 peak at M=N=K=8192 (F32/F16 acc)").
FLOPs = 2MNK per GEMM (the "+C" adds are not counted).

    python bench.py [--gpus N --steps K --warmup W]       # our kernels (default)
    python bench.py --impl reference ...                   # the CPU oracle, bounded sample

Multi-GPU (torchrun, one rank per GPU), default: BASELINE.json north_star's scaling target,
M=N=K=16384 N-sharded (configs[3]: each rank owns a column slab of B and C, A replicated, no
communication in the GEMM phase; strong scaling).  The line reports the GEMM-phase
efficiency T1 / (P * T_P), with T1 the unsharded problem timed on rank 0 in the same run,
plus the NCCL all-gather of C and the fused GEMM + gather kernel (epilogue stores to every
rank's C through symmetric memory).  `--workload batch` runs one independent problem per
GPU instead (configs[4], weak scaling).  Time = max over ranks of the device-timed region.
Inputs are seeded (synth/), uploaded to HBM before the timed region; the
per-step working set (A 128 MB + B 128 MB + C 256/128 MB) exceeds the 126 MB L2.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "GEMM TFLOP/s & % of B200 dense FP16 peak at M=N=K=8192 (F32/F16 acc)"
NOMINAL_F16_DENSE_TFLOPS = 2250.0


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--size", type=int, default=0, help="M = N = K (default 8192; 16384 for the N-shard workload)")
    ap.add_argument("--modes", default="f32,f16")
    ap.add_argument("--config", default="auto", help="kernel configuration (name in CONFIGS)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--sustained-steps", type=int, default=300,
                    help="extra back-to-back steps timed after the main region (power-capped regime); 0 = skip")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="oracle sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-small", action="store_true", help="skip the configs[0]/configs[1] small-shape record")
    ap.add_argument("--workload", choices=["auto", "batch", "nshard"], default="auto",
                    help="auto: nshard with more than one GPU, else one problem; batch: one independent n^3 "
                         "problem per GPU (weak scaling); nshard: one n^3 problem N-sharded over the GPUs "
                         "(strong scaling, BASELINE configs[3])")
    ap.add_argument("--allgather", choices=["auto", "none", "nccl", "fused"], default="auto",
                    help="nshard: auto = time both the NCCL all-gather of the C slabs and the fused "
                         "GEMM + gather kernel (epilogue stores to all ranks' full C buffers through torch "
                         "symmetric memory), each after the GEMM-phase region; none; nccl; fused = the "
                         "fused kernel IS the timed step")
    ap.add_argument("--no-t1", action="store_true", help="nshard: skip the unsharded T1 reference on rank 0")
    ap.add_argument("--dist-backend", default="nccl",
                    help="process-group backend (nccl; 'gloo' plus BENCH_ONE_DEVICE=1 runs every rank on cuda:0 "
                         "-- a 1-GPU check of the multi-rank logic, never a measurement)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.workload == "auto":
        args.workload = "nshard" if world > 1 else "batch"
    if args.size == 0:
        args.size = 16384 if args.workload == "nshard" else 8192
    if args.allgather == "auto":
        args.allgather = "both" if (args.workload == "nshard" and world > 1) else "none"
    return args


def load_peaks():
    """Roofline denominators: MEASURED_PEAKS.json (driver-written), else the
    fallback stated in B200_PROFILING.md (1.59 PFLOP/s burst, 6.65 TB/s)."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            mp = json.load(f)
        return {"tflops": float(mp["bf16_tflops"]), "tflops_sustained": float(mp.get("bf16_tflops_sustained", 0)),
                "hbm_gbs": float(mp["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json bf16_tflops burst; "
                "fp16 dense rate = bf16 rate, nominal ratio 1:1)"}
    except (OSError, KeyError, ValueError):
        return {"tflops": 1590.0, "tflops_sustained": 1400.0, "hbm_gbs": 6650.0,
                "source": "fallback (B200_PROFILING.md: 1.59 PFLOP/s, 6.65 TB/s)"}


class ClockSampler:
    """NVML SM clock + clocks-event reasons, sampled in a thread during the timed region."""
    NAMES = {
        "nvmlClocksEventReasonGpuIdle": "gpu_idle",
        "nvmlClocksEventReasonApplicationsClocksSetting": "applications_clocks_setting",
        "nvmlClocksEventReasonSwPowerCap": "sw_power_cap",
        "nvmlClocksEventReasonHwSlowdown": "hw_slowdown",
        "nvmlClocksEventReasonSyncBoost": "sync_boost",
        "nvmlClocksEventReasonSwThermalSlowdown": "sw_thermal_slowdown",
        "nvmlClocksEventReasonHwThermalSlowdown": "hw_thermal_slowdown",
        "nvmlClocksEventReasonHwPowerBrakeSlowdown": "hw_power_brake_slowdown",
        "nvmlClocksEventReasonDisplayClockSetting": "display_clock_setting",
    }

    def __init__(self, index: int, period_s: float = 0.002):
        self.ok = False
        self.samples = []
        self.reasons = set()
        self.period = period_s
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.bits = {getattr(pynvml, k): v for k, v in self.NAMES.items() if hasattr(pynvml, k)}
            self.ok = True
        except Exception:  # NVML missing: report null clocks
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.bits.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._stop = threading.Event()
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        if self.ok:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons - {"gpu_idle"}), "samples": len(self.samples)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


# ----------------------------------------------------------------------------- oracle arms

def oracle_sample_rate(n: int, modes, budget_s: float, seed: int = 0):
    """Time the CPU oracle, as it stands, on a bounded sample of the workload:
    R rows of every mode's n^3 problem, R calibrated to ~budget_s seconds."""
    import numpy as np
    import oracle
    import synth
    A = synth.uniform_f16(seed, synth.MATRIX_A, n, n)
    B = synth.uniform_f16(seed, synth.MATRIX_B, n, n)
    Cs = {m: (synth.uniform_f32 if m == "f32" else synth.uniform_f16)(seed, synth.MATRIX_C, n, n) for m in modes}
    # OpenMP runs one row per thread, so the cost grows in rounds of `threads`
    # rows: time one full round, then take as many rounds as fit the budget.
    threads = max(1, oracle.num_threads())

    def timed_rounds(k):
        t0 = time.perf_counter()
        for m in modes:
            oracle.gemm(A, B, Cs[m], rows=np.arange(min(n, k * threads)))
        return time.perf_counter() - t0

    # per-call cost (argument marshalling of the n x n inputs) + per-round cost: time one
    # and three rounds (after a warm-up call) and fit both, so the sample fills the budget
    timed_rounds(1)
    t1, t3 = timed_rounds(1), timed_rounds(3)
    t_round = max((t3 - t1) / 2, 1e-6)
    t_call = max(t1 - t_round, 0.0)
    rows = int(min(n, max(1, int(max(budget_s - t_call, t_round) / t_round)) * threads))
    sel = np.linspace(0, n - 1, rows).astype(np.int64)
    t0 = time.perf_counter()
    for m in modes:
        oracle.gemm(A, B, Cs[m], rows=sel)
    dt = time.perf_counter() - t0
    flops = 2.0 * rows * n * n * len(modes)
    return {"value": flops / dt / 1e12, "unit": "TFLOP/s", "cores": oracle.num_threads(), "kind": "oracle",
            "sample": f"{rows} evenly spaced rows of each of the {len(modes)} M=N=K={n} problems "
                      f"({'/'.join(modes)} acc), 2*rows*N*K flop each; {dt:.1f} s host wall clock",
            "seconds": dt, "rows": rows}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import numpy as np
    import oracle
    import synth
    n = args.size
    modes = args.modes.split(",")
    A = synth.uniform_f16(0, synth.MATRIX_A, n, n)
    B = synth.uniform_f16(0, synth.MATRIX_B, n, n)
    Cs = {m: (synth.uniform_f32 if m == "f32" else synth.uniform_f16)(0, synth.MATRIX_C, n, n) for m in modes}
    # size each step so warmup + steps fit in a few minutes (rows run one per
    # OpenMP thread, so a step is a whole number of thread rounds)
    total_budget = 150.0
    per_step = total_budget / max(1, args.steps + args.warmup)
    threads = max(1, oracle.num_threads())

    def timed_rounds(k):
        t0 = time.perf_counter()
        for m in modes:
            oracle.gemm(A, B, Cs[m], rows=np.arange(min(n, k * threads)))
        return time.perf_counter() - t0

    # per-call + per-round cost fitted from one and three rounds (as in oracle_sample_rate)
    timed_rounds(1)
    t1, t3 = timed_rounds(1), timed_rounds(3)
    t_round = max((t3 - t1) / 2, 1e-6)
    t_call = max(t1 - t_round, 0.0)
    # (0.75: margin for the fit, so the whole run stays within ~total_budget)
    rows = int(min(n, max(1, int(max(0.75 * per_step - t_call, t_round) / t_round)) * threads))
    sel = np.linspace(0, n - 1, rows).astype(np.int64)
    for _ in range(args.warmup):
        for m in modes:
            oracle.gemm(A, B, Cs[m], rows=sel)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        for m in modes:
            oracle.gemm(A, B, Cs[m], rows=sel)
    dt = time.perf_counter() - t0
    flops = 2.0 * rows * n * n * len(modes) * args.steps
    value = flops / dt / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded uniform[-1,1) F16 inputs)",
        "config": {"workload": f"M=N=K={n}, F16 inputs, {'+'.join(modes)} accumulate; each step = {rows} "
                               f"sampled rows per mode (bounded CPU sample)", "M": n, "N": n, "K": n},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": oracle.num_threads(), "kind": "oracle",
                         "sample": f"{rows} evenly spaced rows of each M=N=K={n} problem per step"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- our arm

def _time_steps(torch, dist, stream, world, dev, steps, fn):
    """Device time (ms) of `steps` calls of fn() on `stream`, barrier + sync on both sides,
    max over ranks."""
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms


def nshard_scaling(args, g, gdist, dist, torch, A, B, C, slabs, modes, M, N, K, rank, world, dev, stream, tp_ms,
                   make_symmetric_c):
    """SURVEY 8(e) / BASELINE north_star: GEMM-phase strong-scaling efficiency T1 / (P * T_P) at
    the same problem, with T1 = the unsharded GEMMs timed on rank 0 in this run (the other
    ranks idle at a barrier); then the C all-gather over NCCL and the fused GEMM + gather
    kernel, each timed as max over ranks."""
    out = {"P": world, "T_P_ms_per_step": tp_ms, "slab_cols": [n1 - n0 for n0, n1 in slabs]}
    steps = max(3, min(args.steps, 10))
    # full B and C (row-major) assembled from the slabs over NCCL: the NCCL all-gather of C
    # is timed on the way (this IS the gather a user of the sharded GEMM would run)
    gt = {}
    Cfull_rm = {}
    for m in modes:
        gdist.allgather_c(C[m], slabs, layout="slabs")   # warm-up
        gt[m] = _time_steps(torch, dist, stream, world, dev, steps,
                            lambda m=m: gdist.allgather_c(C[m], slabs, layout="slabs")) / steps
        Cfull_rm[m] = gdist.allgather_c(C[m], slabs, layout="rowmajor")
    gbytes = {m: M * N * C[m].element_size() for m in modes}
    out["nccl_allgather"] = {"ms_per_step": sum(gt.values()), "per_mode_ms": gt,
                             "bytes_per_rank_received": {m: gbytes[m] * (world - 1) // world for m in modes},
                             "busbw_gbs": {m: gbytes[m] * (world - 1) / world / (gt[m] * 1e-3) / 1e9 for m in modes},
                             "layout": "slab-major [P][M][N/P] (all_gather_into_tensor)"}
    out["e2e_efficiency_with_nccl_gather"] = None
    # T1: the unsharded problem on rank 0
    if not args.no_t1:
        B_full = gdist.allgather_c(B, slabs, layout="rowmajor")
        torch.cuda.synchronize()
        t1 = None
        if rank == 0:
            with torch.cuda.stream(stream):
                for m in modes:
                    g.gemm_f16(A, B_full, Cfull_rm[m], stream=stream)
            t1 = _time_steps(torch, dist, stream, 1, dev, steps,
                             lambda: [g.gemm_f16(A, B_full, Cfull_rm[m], stream=stream) for m in modes]) / steps
        dist.barrier()
        t = torch.tensor([t1 or 0.0], device=dev, dtype=torch.float64)
        dist.broadcast(t, 0)
        t1 = float(t.item())
        del B_full
        out["T1_ms_per_step"] = t1
        out["gemm_phase_efficiency"] = t1 / (world * tp_ms)
        out["e2e_efficiency_with_nccl_gather"] = t1 / (world * (tp_ms + sum(gt.values())))
        out["T1_how"] = (f"rank 0 alone, the same {M}x{N}x{K} problem unsharded ({'+'.join(modes)} per step), "
                         f"{steps} steps after the sharded region")
    del Cfull_rm
    # fused GEMM + gather (one kernel per mode: epilogue TMA stores to every rank's C)
    if args.allgather in ("both",):
        try:
            Cf = make_symmetric_c()
            from paper_2108_13191_b200 import dist as gd

            def fused_step():
                for m in modes:
                    gd.gemm_nshard_gather(A, B, Cf[m][0], slabs, rank, peer_ptrs=Cf[m][1], stream=stream)
            with torch.cuda.stream(stream):
                fused_step()
            tf = _time_steps(torch, dist, stream, world, dev, steps, fused_step) / steps
            out["fused_gemm_gather"] = {"ms_per_step": tf, "vs_gemm_only": tf / tp_ms}
            if "T1_ms_per_step" in out:
                out["e2e_efficiency_with_fused_gather"] = out["T1_ms_per_step"] / (world * tf)
            del Cf
        except Exception as ex:   # symmetric memory unavailable: report, keep the line
            out["fused_gemm_gather"] = {"error": str(ex)[:200]}
    return out


SMALL_SHAPES = (("configs[0]", 256, "f32"), ("configs[1]", 1024, "f16"))


def small_shapes(g, torch, synth, dev, peaks, reps=20, rounds=5):
    """BASELINE.json configs[0] (256^3 F32 acc) and configs[1] (1024^3 F16 acc): GPU time
    per GEMM from CUDA-graph replay (`reps` launches captured in one graph, median over
    `rounds` replays, CUDA events on the replay stream), so the host enqueue cost of a
    call (~7-11 us) is not counted; against the roofline time of the shape,
    max(2MNK / tensor peak, compulsory bytes / HBM peak), compulsory bytes =
    2(MK + KN) + 2 MN sizeof(C) (C_in read + C_out written).  Inputs fit in L2 here, so
    the HBM term is a floor the kernel need not pay (frac can exceed 1 in principle)."""
    out = {}
    s = torch.cuda.Stream(dev)
    for name, n, mode in SMALL_SHAPES:
        A = torch.from_numpy(synth.uniform_f16(0, synth.MATRIX_A, n, n)).to(dev)
        B = torch.from_numpy(synth.uniform_f16(0, synth.MATRIX_B, n, n)).to(dev)
        C = torch.from_numpy((synth.uniform_f32 if mode == "f32" else synth.uniform_f16)(0, synth.MATRIX_C, n, n)).to(dev)
        with torch.cuda.stream(s):
            for _ in range(3):
                g.gemm_f16(A, B, C, stream=s)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            for _ in range(reps):
                g.gemm_f16(A, B, C, stream=s)
        ts = []
        with torch.cuda.stream(s):   # (replay() launches on the current stream: keep it = s)
            graph.replay()
            torch.cuda.synchronize()
            for _ in range(rounds):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                graph.replay()
                e1.record(s)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) / reps * 1e3)
        us = statistics.median(ts)
        flops = 2.0 * n ** 3
        byts = 2 * (2 * n * n) + 2 * n * n * (4 if mode == "f32" else 2)
        t_tc = flops / (peaks["tflops"] * 1e12) * 1e6
        t_hbm = byts / (peaks["hbm_gbs"] * 1e9) * 1e6
        out[name] = {"M": n, "N": n, "K": n, "mode": mode, "us": round(us, 3), "tflops": round(flops / us / 1e6, 2),
                     "roofline_us": round(max(t_tc, t_hbm), 3), "bound": "hbm" if t_hbm > t_tc else "tensor",
                     "frac": round(max(t_tc, t_hbm) / us, 4), "config": g.pick_config(n, n, n, 0 if mode == "f32" else 1),
                     "how": f"{reps} launches in one CUDA graph, median of {rounds} replays"}
        del graph
    return out


def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    import paper_2108_13191_b200 as g

    rank, world, local = dist_env()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (the product path has no CPU fallback)")
    if os.environ.get("BENCH_ONE_DEVICE") == "1":
        local = 0   # (logic check only: all ranks share one GPU)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 and args.dist_backend != "nccl":
        dist.init_process_group(args.dist_backend)
    elif world > 1:
        # NCCL's init log (rank count, transports: NVLS / P2P over NVLink) goes to stderr, so the
        # driver can check how many ranks the communicator really spans
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=dev)
    g.load_library()

    n = args.size
    M = N = K = n
    modes = args.modes.split(",")
    nshard = args.workload == "nshard"
    if nshard:
        from paper_2108_13191_b200 import dist as gdist
        seed = 0
        slabs = gdist.column_slabs(N, world, align=8)
        n0, n1 = slabs[rank]
    else:
        seed = rank  # one independent problem per GPU
        n0, n1 = 0, N
    nr = n1 - n0
    A_h = synth.uniform_f16(seed, synth.MATRIX_A, M, K)
    B_h = synth.uniform_f16(seed, synth.MATRIX_B, K, N, col_lo=n0, col_hi=n1)
    C_h = {"f32": synth.uniform_f32(seed, synth.MATRIX_C, M, N, col_lo=n0, col_hi=n1),
           "f16": synth.uniform_f16(seed, synth.MATRIX_C, M, N, col_lo=n0, col_hi=n1)}
    A = torch.from_numpy(A_h).to(dev)
    B = torch.from_numpy(B_h).to(dev)
    C = {m: torch.from_numpy(C_h[m]).to(dev) for m in modes}
    fused = nshard and args.allgather == "fused"
    Cfull = {}

    def make_symmetric_c():
        out = {}
        # every rank holds the full C (identical C_in); each step's kernel writes its
        # slab into all ranks' buffers (peer pointers from symmetric memory)
        for m in modes:
            full_h = (synth.uniform_f32 if m == "f32" else synth.uniform_f16)(seed, synth.MATRIX_C, M, N)
            if world > 1:
                t, peers, hdl = gdist.symmetric_c_buffer(M, N, torch.float32 if m == "f32" else torch.float16)
                t.copy_(torch.from_numpy(full_h))
            else:
                t, peers, hdl = torch.from_numpy(full_h).to(dev), [], None
            out[m] = (t, peers, hdl)
        if world > 1:
            torch.cuda.synchronize()
            dist.barrier()
        return out

    if fused:
        Cfull = make_symmetric_c()
    stream = torch.cuda.Stream(dev)
    flops = 2.0 * M * nr * K          # this rank's FLOPs per GEMM
    job_flops = 2.0 * M * N * K * (1 if nshard else world)   # whole job, per GEMM mode

    def step(ev=None, trace=None):
        for i, m in enumerate(modes):
            if ev is not None:
                ev[m][0].record(stream)
            if fused:
                gdist.gemm_nshard_gather(A, B, Cfull[m][0], slabs, rank, peer_ptrs=Cfull[m][1], stream=stream)
            elif i == 0 and trace is not None:
                g.gemm_f16(A, B, C[m], stream=stream, config=args.config, trace=trace)
            else:
                g.gemm_f16(A, B, C[m], stream=stream, config=args.config)
            if ev is not None:
                ev[m][1].record(stream)

    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    ev = {m: [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)] for m in modes}
    tr_in = None if fused else torch.zeros(512, dtype=torch.int64, device=dev)
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    launches = 0
    with ClockSampler(local) as clk:
        t_start.record(stream)
        for s in range(args.steps):
            # the middle step's first GEMM records CTA 0's per-tile clock64 / globaltimer (one
            # thread, a few stores per tile): the SM clock the timed kernels actually ran at
            step({m: ev[m][s] for m in modes}, trace=tr_in if s == args.steps // 2 else None)
            launches += len(modes) * g.last_launches()
        t_end.record(stream)
        torch.cuda.synchronize()
    elapsed_ms = t_start.elapsed_time(t_end)
    if world > 1:
        dist.barrier()
        t = torch.tensor([elapsed_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    per_mode_ms = {m: statistics.mean(ev[m][s][0].elapsed_time(ev[m][s][1]) for s in range(args.steps)) for m in modes}
    value = job_flops * len(modes) * args.steps / (elapsed_ms * 1e-3) / 1e12

    peaks = load_peaks()
    mode_stats = {m: {"tflops": flops / (per_mode_ms[m] * 1e-3) / 1e12, "ms": per_mode_ms[m],
                      "frac_of_2250": flops / (per_mode_ms[m] * 1e-3) / 1e12 / NOMINAL_F16_DENSE_TFLOPS,
                      "frac_of_measured_peak": flops / (per_mode_ms[m] * 1e-3) / 1e12 / peaks["tflops"],
                      "config": g.pick_config(M, N, K, 0 if m == "f32" else 1) if args.config == "auto"
                      else g.CONFIGS[args.config]} for m in modes}
    dom = max(modes, key=lambda m: per_mode_ms[m])
    achieved = mode_stats[dom]["tflops"]
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                traffic = json.load(f).get(f"{n}_{dom}")
        except (OSError, ValueError):
            traffic = None

    # --------------------------------------------------------- SM clock seen by the kernel itself
    # NVML's clock reading lags over a ~50 ms window; the traced launch inside the timed region
    # (middle step, first mode) gives clock64 / globaltimer of CTA 0's MMA warp per tile.
    kernel_clock = None
    if tr_in is not None:
        try:
            t = tr_in.cpu().numpy().reshape(64, 8)
            ghz = [t[i, 7] / (t[i, 2] - t[i, 0]) for i in range(60) if t[i, 0] and t[i, 2] > t[i, 0] and t[i, 7]]
            if ghz:
                kernel_clock = {"sm_mhz_median": round(1000 * float(statistics.median(ghz)), 1),
                                "sm_mhz_min": round(1000 * float(min(ghz)), 1),
                                "sm_mhz_max": round(1000 * float(max(ghz)), 1), "tiles": len(ghz),
                                "how": f"clock64/globaltimer of CTA 0's MMA warp per tile, traced in place in timed "
                                       f"step {args.steps // 2} ({modes[0]} GEMM)"}
        except Exception as ex:  # tracing is diagnostic only
            kernel_clock = {"error": str(ex)[:120]}

    # the same kernel against the dense tensor peak at the SM clock it actually ran at (148 SMs x
    # 8192 dense FP16 FLOP/clk; B200_PROFILING.md unit counts): how much of the gap to the
    # nominal peak is the power-capped clock rather than the kernel
    clock_adjusted = None
    if kernel_clock and "sm_mhz_median" in kernel_clock and modes[0] == dom:
        at_clock = 148 * 8192 * kernel_clock["sm_mhz_median"] * 1e6 / 1e12
        clock_adjusted = {"sm_mhz": kernel_clock["sm_mhz_median"], "peak_at_clock_tflops": at_clock,
                          "frac": achieved / at_clock,
                          "how": "achieved / (148 SMs x 8192 FLOP/clk x the traced SM clock of a timed launch)"}

    # --------------------------------------------------------- sustained (power-capped) regime
    # The main region (~50 ms) is a burst: the board has not yet settled at its
    # power cap and NVML's clock reading lags.  Run the same steps back to back for
    # longer and report them against the driver's SUSTAINED peak.
    sustained = None
    if args.sustained_steps > 0:
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        with ClockSampler(local, period_s=0.005) as sclk:
            s0.record(stream)
            for _ in range(args.sustained_steps):
                step()
            s1.record(stream)
            torch.cuda.synchronize()
        s_ms = s0.elapsed_time(s1)
        if world > 1:
            t = torch.tensor([s_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            s_ms = float(t.item())
        s_val = job_flops * len(modes) * args.sustained_steps / (s_ms * 1e-3) / 1e12
        sustained = {"value": s_val, "unit": "TFLOP/s", "steps": args.sustained_steps, "ms_per_step": s_ms / args.sustained_steps,
                     "peak": peaks["tflops_sustained"], "frac_of_sustained_peak": s_val / peaks["tflops_sustained"] if peaks["tflops_sustained"] else None,
                     "clocks": sclk.summary(),
                     "note": "same steps back to back for longer, after the main region; peak = MEASURED_PEAKS "
                             "bf16_tflops_sustained (cuBLAS, 4 s back to back)"}

    # --------------------------------------------------------- e2e through the host-buffer C ABI
    e2e = None
    if not args.no_e2e:
        hA = torch.from_numpy(A_h).pin_memory()
        hB = torch.from_numpy(B_h).pin_memory()
        hC = {m: torch.from_numpy(C_h[m].copy()).pin_memory() for m in modes}
        dC = {m: torch.empty_like(C[m]) for m in modes}
        dA = torch.empty_like(A)
        dB = torch.empty_like(B)

        e2e_launches = [0]

        def e2e_step():
            # the step's GEMMs share A and B: the first call copies them in, the
            # others reuse them from dA / dB (hA = hB = None: resident operands)
            for i, m in enumerate(modes):
                g.gemm_f16_host(hA if i == 0 else None, hB if i == 0 else None, hC[m], dA, dB, dC[m],
                                stream=stream)
                e2e_launches[0] += g.last_launches()
        e2e_step()
        torch.cuda.synchronize()
        e2e_launches[0] = 0
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([e_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        h2d = A_h.nbytes + B_h.nbytes + sum(C_h[m].nbytes for m in modes)
        d2h = sum(C_h[m].nbytes for m in modes)
        e2e = {"value": job_flops * len(modes) * args.e2e_steps / (e_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": args.e2e_steps,
               "ms_per_step": e_ms / args.e2e_steps,
               "path": "gemm_f16_host (C ABI): pinned host A,B,C -> row-block pipeline of H2D / GEMM / D2H "
                       "on three streams, per mode; A and B copied once per step (the second call "
                       "passes them as resident)",
               "gpu_launches": e2e_launches[0]}

    # --------------------------------------------------------- optional NCCL all-gather of C (nshard)
    gather = None
    if fused:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        gather = {"mode": "fused", "ms_per_step": None,
                  "bytes_gathered_per_step": sum(M * N * Cfull[m][0].element_size() for m in modes),
                  "note": "the gather is inside the timed GEMM kernels (epilogue TMA stores to all ranks' C)"}
    scaling_block = None
    if nshard and world > 1:
        scaling_block = nshard_scaling(args, g, gdist, dist, torch, A, B, C, slabs, modes, M, N, K, rank, world, dev,
                                       stream, elapsed_ms / args.steps, make_symmetric_c)

    # --------------------------------------------------------- sampled parity of this launch config
    parity = None
    if rank == 0 and not args.no_parity:
        import oracle
        rows = synth.sample_rows(M, tile_m=256, n_random=0)[:: max(1, M // 256 // 8)][:12]
        parity = {"rows": int(len(rows))}
        ok = True
        for m in modes:
            Cm = torch.from_numpy(C_h[m]).to(dev)
            g.gemm_f16(A, B, Cm, stream=stream, config=args.config)
            torch.cuda.synchronize()
            got = Cm[torch.from_numpy(rows).to(dev)].cpu().numpy().astype(np.float64)
            ex, _ = oracle.gemm(A_h, B_h, C_h[m], rows=rows)
            err = got - ex
            rel = float(np.linalg.norm(err) / np.linalg.norm(ex))
            parity[m] = {"rel_fro": rel, "max_abs": float(np.abs(err).max())}
            if m == "f32":
                bound = 1e-3 * np.sqrt(K) * float(np.abs(A_h.astype(np.float32)).max()) * float(np.abs(B_h.astype(np.float32)).max())
                ok &= rel <= 1e-5 and parity[m]["max_abs"] <= bound
            else:
                ok &= rel <= 2e-3
        parity["pass"] = bool(ok)

    small = None
    if rank == 0 and not args.no_small:
        small = small_shapes(g, torch, synth, dev, load_peaks())

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_sample_rate(n, modes, args.cpu_seconds)
        cpu.pop("seconds", None)
        cpu.pop("rows", None)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if nshard else "weak", "vs_baseline": None, "dtype": "f16",
            "data": "synthetic (seeded uniform[-1,1) inputs rounded to F16; C_in uniform F32/F16)",
            "config": {"workload": f"M=N=K={n} C+=A.B, F16 A/B row-major; one F32-acc and one F16-acc GEMM "
                                   f"per step" if len(modes) == 2 else f"M=N=K={n}, {modes[0]} acc",
                       "M": M, "N": N, "K": K, "modes": modes,
                       "kernel_config": args.config,
                       "l2": "inputs larger than L2 (A 128 MB + B 128 MB + C 256/128 MB per step > 126 MB)",
                       "parallelism": ("single GPU" if world == 1 else
                                       f"N-shard x{world}: A replicated, B/C column slabs" if nshard else
                                       f"batch-one-per-GPU x{world} (no collective)"),
                       "workload_kind": args.workload},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peaks["tflops"], "unit": "TFLOP/s",
                         "frac": achieved / peaks["tflops"], "traffic": traffic, "kernel": f"gemm {dom}-acc",
                         "algorithmic_flops_per_launch": flops,
                         "algorithmic_bytes_per_launch": 2 * (M * K + K * nr) + 2 * M * nr * (4 if dom == "f32" else 2),
                         "peak_source": peaks["source"],
                         "frac_of_nominal_2250": achieved / NOMINAL_F16_DENSE_TFLOPS,
                         "clock_adjusted": clock_adjusted},
            "modes": mode_stats,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "sustained": sustained,
            "clocks": dict(clk.summary(), kernel_measured=kernel_clock,
                           regime="burst: ~50 ms timed window after warm-up; see 'sustained' for the "
                                  "power-capped regime",
                           note="NVML sm_mhz is sampled every 2 ms but lags over a 50 ms window; "
                                "kernel_measured is the SM clock of one of the timed GEMMs, traced in place "
                                "(sw_power_cap shows up in the longer 'sustained' window)"),
            "parity": parity,
            "small_shapes": small,
            "allgather": gather,
            "nshard_scaling": scaling_block,
            "comm": ({"backend": dist.get_backend(), "nranks": dist.get_world_size(),
                      "nccl_version": ".".join(str(x) for x in torch.cuda.nccl.version()),
                      "init_log": "NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT on stderr"} if world > 1 else None),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()   # rank 0 may still be on its CPU parity check
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

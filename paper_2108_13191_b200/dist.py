"""Multi-GPU plumbing for the GEMM (BASELINE.json north_star):

* N-sharding: rank r owns the column slab B[:, n_r0:n_r1] and C[:, n_r0:n_r1]
  (A replicated).  Each rank runs one independent gemm_f16 on its slab -- no
  communication in the compute phase.  `allgather_c` optionally gathers the C
  slabs over NCCL (torch.distributed all_gather_into_tensor on NVLink/NVSwitch).
* Batch-one-per-GPU: independent problems are distributed round-robin over ranks
  (no collective at all).

The paper itself is single-GPU (Sec. 4); this is the B200
box's data decomposition of the same C = AB + C.  Host logic only:
every FLOP runs in libgemm_f16.so via `paper_2108_13191_b200.gemm_f16`.
"""
from __future__ import annotations

from typing import Callable, Sequence


def column_slabs(N: int, world: int, align: int = 8):
    """Split [0, N) into `world` contiguous column slabs, as equal as possible,
    every internal boundary a multiple of `align` elements (so each slab's first
    column keeps 16-byte TMA alignment for F16 B and F16/F32 C).  Returns a list
    of (n0, n1); trailing ranks may get empty slabs when N is tiny."""
    if world <= 0:
        raise ValueError("world must be positive")
    if N < 0:
        raise ValueError("N must be non-negative")
    units = -(-N // align)                     # ceil(N / align) alignment units
    base, extra = divmod(units, world)
    out = []
    u = 0
    for r in range(world):
        cnt = base + (1 if r < extra else 0)
        n0 = min(N, u * align)
        n1 = min(N, (u + cnt) * align)
        out.append((n0, n1))
        u += cnt
    return out


def gemm_nshard(A, B_r, C_r, compute: Callable | None = None, **kw):
    """This rank's share of an N-sharded C += A.B: C_r += A @ B_r (slab-local).

    A: (M, K) F16 replicated; B_r: (K, n_r) F16; C_r: (M, n_r) F32/F16.
    `compute` defaults to the CUDA kernel; tests may inject another callable with
    the same signature to exercise the host logic on CPU."""
    if compute is None:
        from . import gemm_f16 as compute
    if B_r.shape[1] == 0:
        return C_r
    return compute(A, B_r, C_r, **kw)


def allgather_c(C_r, n_slabs: Sequence[tuple[int, int]], group=None, layout: str = "rowmajor"):
    """Gather every rank's C slab.  Slabs are padded to the widest slab so one
    all_gather_into_tensor (NCCL) moves them; result is either the slab-major
    stack [P, M, w_max] (layout="slabs") or the row-major M x N matrix
    (layout="rowmajor", one extra device copy)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    if len(n_slabs) != world:
        raise ValueError("n_slabs must have one entry per rank")
    M = C_r.shape[0]
    w_max = max(n1 - n0 for n0, n1 in n_slabs)
    send = C_r
    if C_r.shape[1] != w_max or not C_r.is_contiguous():
        send = torch.zeros((M, w_max), dtype=C_r.dtype, device=C_r.device)
        send[:, : C_r.shape[1]] = C_r
    out = torch.empty((world, M, w_max), dtype=C_r.dtype, device=C_r.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, send, group=group)
    else:  # gloo (CPU tests): list form
        parts = list(out.unbind(0))
        dist.all_gather(parts, send, group=group)
    if layout == "slabs":
        return out
    if layout != "rowmajor":
        raise ValueError(layout)
    return torch.cat([out[r, :, : n1 - n0] for r, (n0, n1) in enumerate(n_slabs)], dim=1)


def my_problems(n_problems: int, rank: int, world: int):
    """Indices of the independent problems this rank runs (round-robin)."""
    return list(range(rank, n_problems, world))


def gemm_batched_one_per_gpu(problems, rank: int, world: int, compute: Callable | None = None, **kw):
    """Run this rank's share of a list of independent (A, B, C) problems in place."""
    if compute is None:
        from . import gemm_f16 as compute
    done = []
    for i in my_problems(len(problems), rank, world):
        A, B, C = problems[i]
        compute(A, B, C, **kw)
        done.append(i)
    return done


def gemm_nshard_gather(A, B_r, C_full, n_slabs, rank: int, peer_ptrs=(), **kw):
    """Fused N-shard + all-gather (one kernel): this rank computes its column slab
    of C_full (C_in read from its own C_full) and its epilogue stores each finished
    tile into C_full and into every peer's C_full (`peer_ptrs`: device addresses
    of the other ranks' full C buffers, e.g. from `symmetric_c_buffer`).  After
    every rank's kernel has completed (synchronise, then a cross-rank barrier),
    every C_full holds the whole result -- the gather overlapped the math instead
    of following it."""
    from . import gemm_f16_gather
    n0, n1 = n_slabs[rank]
    if n1 == n0:
        return C_full
    return gemm_f16_gather(A, B_r, C_full, n0, peers=peer_ptrs, **kw)


def symmetric_c_buffer(M: int, N: int, dtype, group=None):
    """Allocate this rank's full C in torch symmetric memory and return
    (tensor, [peer device addresses of the other ranks' buffers], handle).
    Needs NVLink-connected GPUs in one node (CUDA IPC); the handle's barrier()
    orders readers after all ranks' writers."""
    import torch
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm_mem

    t = symm_mem.empty((M, N), dtype=dtype, device=torch.device("cuda", torch.cuda.current_device()))
    hdl = symm_mem.rendezvous(t, group=group if group is not None else dist.group.WORLD)
    me = hdl.rank
    peers = [int(p) for r, p in enumerate(hdl.buffer_ptrs) if r != me]
    return t, peers, hdl

"""Worker of tests/test_dist_gpu.py, one process per GPU under torchrun (NCCL): the
N-sharded C += A.B, its NCCL all-gather and the fused GEMM + gather kernel
(gemm_f16_gather storing into every rank's symmetric-memory C) against the CPU oracle.
Rank 0 writes a JSON verdict to argv[1]."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np
import torch
import torch.distributed as dist

import oracle
import synth
import paper_2108_13191_b200 as g
from paper_2108_13191_b200 import dist as gdist
from parity import check


def main(out_path):
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    res = {"world": world, "nranks": dist.get_world_size()}
    M, N, K = 1000, 2056, 1536          # ragged M, slabs of 8-column multiples
    slabs = gdist.column_slabs(N, world, align=8)
    n0, n1 = slabs[rank]
    for acc in ("f32", "f16"):
        A, B, C = synth.problem(M, N, K, acc, seed=21)
        dA = torch.from_numpy(A).to(dev)
        B_r = torch.from_numpy(np.ascontiguousarray(B[:, n0:n1])).to(dev)
        C_r = torch.from_numpy(np.ascontiguousarray(C[:, n0:n1])).to(dev)
        gdist.gemm_nshard(dA, B_r, C_r)
        full = gdist.allgather_c(C_r, slabs, layout="rowmajor")
        # fused: every rank's symmetric C receives every slab from the owners' epilogues
        t, peers, hdl = gdist.symmetric_c_buffer(M, N, torch.float32 if acc == "f32" else torch.float16)
        t.copy_(torch.from_numpy(C))
        torch.cuda.synchronize()
        dist.barrier()
        gdist.gemm_nshard_gather(dA, B_r, t, slabs, rank, peer_ptrs=peers)
        torch.cuda.synchronize()
        hdl.barrier()
        dist.barrier()
        if rank == 0:
            ex, _ = oracle.gemm(A, B, C)
            s1 = check(full.cpu().numpy(), ex, A, B, acc, K, f"nshard + NCCL gather {acc}")
            s2 = check(t.cpu().numpy(), ex, A, B, acc, K, f"fused gather {acc}")
            bits = torch.int32 if acc == "f32" else torch.int16
            same = bool(torch.equal(full.view(bits), t.view(bits)))
            res[acc] = {"nccl_rel_fro": s1["rel_fro"], "fused_rel_fro": s2["rel_fro"], "bitwise_equal": same}
        dist.barrier()
    if rank == 0:
        with open(out_path, "w") as f:
            json.dump(res, f)
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])

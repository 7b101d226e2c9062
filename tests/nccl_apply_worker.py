"""torchrun worker for tests/test_gpu_hardening.py (not collected by pytest).

Initialises NCCL (one process per GPU), shards a seeded matrix by owners, and runs
``distributed.apply_sharded`` with its default CUDA apply (NCCL broadcast of C/S from
rank 0, then the pipeline kernel on the local shard). Each rank writes its shard and
range to OUT_DIR for the parent test to reassemble and compare with the oracle.
"""

from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    out_dir = sys.argv[1]
    m, n, k = (int(x) for x in sys.argv[2:5])
    side, order, kind, fast = sys.argv[5], sys.argv[6], sys.argv[7], sys.argv[8] == "fast"
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    try:
        from paper_2412_01852_b200 import generate_sequence, make_inputs
        from paper_2412_01852_b200.distributed import apply_sharded, owner_shard

        A, seq = make_inputs(m, n, k, 21)
        if side == "left":
            seq = generate_sequence(m, k, 22)
        owners = n if side == "left" else m
        o0, o1 = owner_shard(owners, world, rank)
        part = A[:, o0:o1] if side == "left" else A[o0:o1, :]
        dA = torch.from_numpy(np.asfortranarray(part)).to(dev)
        assert dA.stride(0) == 1
        if rank == 0:
            C = torch.from_numpy(seq.C).to(dev)
            S = torch.from_numpy(seq.S).to(dev)
        else:  # received through the NCCL broadcast
            C = torch.full(seq.C.shape, float("nan"), dtype=torch.float64, device=dev).t().contiguous().t()
            S = torch.full(seq.S.shape, float("nan"), dtype=torch.float64, device=dev).t().contiguous().t()
        apply_sharded(dA, C, S, kind=kind, fast=fast, side=side, order=order)
        torch.cuda.synchronize(dev)
        np.save(os.path.join(out_dir, f"rank{rank}.npy"), dA.cpu().numpy())
        np.save(os.path.join(out_dir, f"range{rank}.npy"), np.array([o0, o1]))
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

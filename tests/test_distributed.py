"""Multi-rank host logic on CPU (gloo, world_size 2): owner sharding + C/S broadcast.
The per-rank compute is the CPU oracle (the GPU kernel is covered by the -m gpu
tests); the check is that the sharded result equals the unsharded one bit for bit —
the "GPU-count invariance" property of SURVEY §4/§8(e)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle
        from paper_2412_01852_b200 import generate_sequence, make_inputs
        from paper_2412_01852_b200.distributed import apply_sharded, owner_shard

        m, n, k, side, order, kind = case
        A, seq = make_inputs(m, n, k, 3)
        if side == "left":
            seq = generate_sequence(m, k, 4)
        owners = n if side == "left" else m
        o0, o1 = owner_shard(owners, world, rank)
        local = np.asfortranarray(A[:, o0:o1] if side == "left" else A[o0:o1, :])
        # only rank 0 holds the real coefficients; the others receive them
        if rank == 0:
            C = torch.from_numpy(seq.C.copy())
            S = torch.from_numpy(seq.S.copy())
        else:
            C = torch.zeros(seq.C.shape, dtype=torch.float64)
            S = torch.zeros(seq.S.shape, dtype=torch.float64)

        def cpu_apply(A_local, cs, kind_, fast, side_, order_):
            Cb, Sb = (t.numpy() for t in cs)
            oracle.apply_naive(A_local, Cb, Sb, side=side_.value, order=order_.value, kind=kind_.value, fast=fast)

        apply_sharded(local, C, S, kind=kind, side=side, order=order, apply_fn=cpu_apply)
        np.save(os.path.join(out_dir, f"rank{rank}.npy"), local)
        np.save(os.path.join(out_dir, f"range{rank}.npy"), np.array([o0, o1]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [
    (300, 40, 12, "right", "forward", "rotation"),
    (70, 200, 9, "left", "reverse", "reflector"),
    (129, 33, 20, "right", "reverse", "rotation"),
])
def test_sharded_equals_unsharded_gloo(tmp_path, case, oracle_mod):
    from paper_2412_01852_b200 import generate_sequence, make_inputs

    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), case, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    m, n, k, side, order, kind = case
    A, seq = make_inputs(m, n, k, 3)
    if side == "left":
        seq = generate_sequence(m, k, 4)
    ref = A.copy(order="F")
    oracle_mod.apply_naive(ref, seq.C, seq.S, side=side, order=order, kind=kind)
    got = np.empty_like(ref)
    for r in range(world):
        o0, o1 = np.load(tmp_path / f"range{r}.npy")
        part = np.load(tmp_path / f"rank{r}.npy")
        if side == "left":
            got[:, o0:o1] = part
        else:
            got[o0:o1, :] = part
    assert np.array_equal(np.ascontiguousarray(ref).view(np.uint64), np.ascontiguousarray(got).view(np.uint64))

"""Multi-GPU application: owners sharded across ranks, one broadcast of C/S.

Rows are independent for right-side application and columns for the left side
(the reference parallelises exactly this way over threads: partition_rows /
_run_row_ranges, blocking.py:178-202, 518-526; "the threads apply the same
rotations to different rows"). Each rank owns a contiguous
shard of owners in units of the CTA tile (``workloads.shard_range``); rank 0's
C/S are broadcast once (NCCL over NVLink/NVSwitch with backend "nccl", gloo on
CPU for tests). There is no other communication and no data-path collective.

One process per GPU; launched by ``torch.distributed.run``.
"""

from __future__ import annotations

from .core import Order, Side, TransformKind, _as_enum
from .workloads import shard_range

TILE_OWNERS = 64  # rows (right) / columns (left) per CTA tile of the pipeline kernel


def owner_shard(total_owners: int, world: int, rank: int):
    """[o0, o1) of the owners this rank holds (tile-aligned, leftovers to the last)."""
    return shard_range(total_owners, world, rank, align=TILE_OWNERS)


def broadcast_sequence(C, S, src: int = 0, group=None):
    """Broadcast rank ``src``'s C and S (torch tensors of identical shape/dtype on
    every rank; contents only matter on src) in place; returns (C, S)."""
    import torch.distributed as dist  # noqa: PLC0415

    dist.broadcast(C, src=src, group=group)
    dist.broadcast(S, src=src, group=group)
    return C, S


def apply_sharded(A_local, C, S, kind=TransformKind.ROTATION, fast: bool = False, side=Side.RIGHT,
                  order=Order.FORWARD, src: int = 0, group=None, apply_fn=None) -> None:
    """Broadcast C/S from ``src`` then transform this rank's shard in place.

    ``A_local`` is this rank's rows (right side) or columns (left side) of A as a
    column-major tensor; C/S are the full (len-1) x k arrays (len is unsharded).
    ``apply_fn(A_local, (C, S), kind, fast, side, order)`` defaults to the CUDA path
    (``apply_device``); tests substitute the CPU oracle to exercise the host logic.
    """
    kind = _as_enum(kind, TransformKind, "kind")
    side = _as_enum(side, Side, "side")
    order = _as_enum(order, Order, "order")
    broadcast_sequence(C, S, src=src, group=group)
    if apply_fn is None:
        from .apply import apply_device  # noqa: PLC0415

        apply_device(A_local, (C, S), kind=kind, fast=fast, side=side, order=order)
    else:
        apply_fn(A_local, (C, S), kind, fast, side, order)

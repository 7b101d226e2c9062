"""Multi-GPU application: owners sharded across ranks, one broadcast of C/S.

Rows are independent for right-side application and columns for the left side
(the reference parallelises exactly this way over threads: partition_rows /
_run_row_ranges, blocking.py:178-202, 518-526; "the threads apply the same
rotations to different rows"). Each rank owns a contiguous
shard of owners in units of the CTA tile (``owner_shard``); rank ``src``'s C/S are
broadcast (NCCL over NVLink/NVSwitch with backend "nccl", gloo on CPU for tests).
There is no other communication and no data-path collective: the shards never
exchange matrix data, so the result on every rank is bit-identical to the same
rows of a single-GPU application in strict mode (GPU-count invariance).

One process per GPU, launched by ``torch.distributed.run``:

* ``owner_shard(total, world, rank)``      which rows (right) / columns (left) a rank holds
* ``ShardedApplier``                        a rank's resident shard + packed sequence; ``step()``
                                            = broadcast C/S, repack, apply (what ``bench.py``
                                            times at N > 1, each phase on its own events)
* ``apply_sharded(A_local, C, S, ...)``     one-shot form of the same step
"""

from __future__ import annotations

from .core import Order, Side, TransformKind, _as_enum
from .workloads import shard_range

TILE_OWNERS = 64  # rows (right) / columns (left) per CTA tile of the pipeline kernel


def owner_shard(total_owners: int, world: int, rank: int):
    """[o0, o1) of the owners this rank holds (tile-aligned, leftovers to the last)."""
    return shard_range(total_owners, world, rank, align=TILE_OWNERS)


def _dense_view(X):
    """A contiguous view of X's storage (X itself, or its transpose for the column-major
    C/S the library uses), or None when X is not dense in either order."""
    if X.is_contiguous():
        return X
    if X.dim() == 2 and X.t().is_contiguous():
        return X.t()
    return None


def broadcast_sequence(C, S, src: int = 0, group=None):
    """Broadcast rank ``src``'s C and S (torch tensors of identical shape, dtype and
    strides on every rank; contents only matter on src) in place; returns (C, S).
    Column-major C/S are sent as their dense storage (NCCL needs contiguous buffers)."""
    import torch.distributed as dist  # noqa: PLC0415

    for X in (C, S):
        view = _dense_view(X)
        if view is not None:
            dist.broadcast(view, src=src, group=group)
        else:
            tmp = X.contiguous()
            dist.broadcast(tmp, src=src, group=group)
            X.copy_(tmp)
    return C, S


class ShardedApplier:
    """One rank's part of a sharded application with A resident in HBM.

    ``A_local`` is this rank's rows (right side) or columns (left side) of A as a
    column-major CUDA tensor; ``C``/``S`` are full (len-1) x k CUDA tensors on every
    rank (their contents matter on ``src`` only until the first broadcast). The
    coefficient records are packed into a persistent workspace
    (``PackedSequence``, the reference's prepacked tier blocking.py:479-515)."""

    def __init__(self, A_local, C, S, kind=TransformKind.ROTATION, fast: bool = False, side=Side.RIGHT,
                 order=Order.FORWARD, src: int = 0, group=None, distributed: bool | None = None):
        from .apply import PackedSequence  # noqa: PLC0415

        self.kind = _as_enum(kind, TransformKind, "kind")
        self.side = _as_enum(side, Side, "side")
        self.order = _as_enum(order, Order, "order")
        self.fast = bool(fast)
        self.A, self.C, self.S = A_local, C, S
        self.src, self.group = src, group
        if distributed is None:
            import torch.distributed as dist  # noqa: PLC0415

            distributed = dist.is_available() and dist.is_initialized()
        self.distributed = distributed
        self.broadcast()
        self.packed = PackedSequence((C, S), tuple(A_local.shape), kind=self.kind, side=self.side, order=self.order,
                                     dtype=A_local.dtype, device=A_local.device, fast_only=self.fast)

    def broadcast(self) -> None:
        if self.distributed:
            broadcast_sequence(self.C, self.S, src=self.src, group=self.group)

    def pack(self) -> None:
        self.packed.pack((self.C, self.S))

    def apply(self) -> None:
        self.packed.apply(self.A, fast=self.fast)

    def step(self, events=None) -> None:
        """Broadcast, repack, apply. ``events`` (4 CUDA events) are recorded on the
        current stream before the broadcast and after each phase."""
        import torch  # noqa: PLC0415

        stream = torch.cuda.current_stream(self.A.device)
        if events is not None:
            events[0].record(stream)
        self.broadcast()
        if events is not None:
            events[1].record(stream)
        self.pack()
        if events is not None:
            events[2].record(stream)
        self.apply()
        if events is not None:
            events[3].record(stream)


def apply_sharded(A_local, C, S, kind=TransformKind.ROTATION, fast: bool = False, side=Side.RIGHT,
                  order=Order.FORWARD, src: int = 0, group=None, apply_fn=None) -> None:
    """Broadcast C/S from ``src`` then transform this rank's shard in place.

    Default (CUDA tensors): one ``ShardedApplier`` step on the device. ``apply_fn(A_local,
    (C, S), kind, fast, side, order)`` substitutes another apply after the same broadcast
    (the gloo tests run the CPU oracle there to exercise the host logic without a GPU).
    """
    kind = _as_enum(kind, TransformKind, "kind")
    side = _as_enum(side, Side, "side")
    order = _as_enum(order, Order, "order")
    if apply_fn is None:
        ShardedApplier(A_local, C, S, kind=kind, fast=fast, side=side, order=order, src=src, group=group).apply()
        return
    broadcast_sequence(C, S, src=src, group=group)
    apply_fn(A_local, (C, S), kind, fast, side, order)

"""BASELINE.json workloads (configs 1-5) and their seeded synthetic inputs.

There is no public dataset for this path: the paper sweeps synthetic m = n
matrices with k = 180 and the reference generates its inputs
from Philox seeds (verification.py:102-105). Generation follows SURVEY §8(d):

1. 512^2, k=64, fp64, right/forward        exactly make_inputs(512, 512, 64, 0)
2. 4096^2, k=192, fp64, right/forward      exactly make_inputs(4096, 4096, 192, 0)
3. 65536x2048, k=256, fp64, right/forward  make_inputs(65536, 2048, 256, 0); row-sharded
4. 8192^2, k=128, fp32, right/forward      A = Philox(0).uniform(-1, 1) -> f32,
                                           theta = Philox(1).uniform(0, 2pi) (f64 cos/sin -> f32)
5. 16384^2, k=96, fp64, left/reverse       A = Philox(0).standard_normal, entries i > j+1
                                           zeroed (upper Hessenberg); theta = Philox(1).uniform
                                           (-pi/2, pi/2) of shape (m-1, k); column-sharded
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import Order, Side, flops_applied, generate_sequence


@dataclass(frozen=True)
class Workload:
    index: int
    m: int
    n: int
    k: int
    dtype: type
    side: Side
    order: Order
    description: str

    @property
    def length(self) -> int:
        return self.m if self.side is Side.LEFT else self.n

    @property
    def owners(self) -> int:
        return self.n if self.side is Side.LEFT else self.m

    @property
    def flops(self) -> float:
        return flops_applied(self.m, self.n, self.k, self.side)

    @property
    def itemsize(self) -> int:
        return np.dtype(self.dtype).itemsize

    def algorithmic_bytes(self) -> float:
        """Read A once + write A once + read C and S once."""
        return 2.0 * self.m * self.n * self.itemsize + 2.0 * (self.length - 1) * self.k * self.itemsize

    def name(self) -> str:
        return (f"config{self.index}: m={self.m} n={self.n} k={self.k} "
                f"{np.dtype(self.dtype).name} {self.side.value}/{self.order.value}")


WORKLOADS = {
    1: Workload(1, 512, 512, 64, np.float64, Side.RIGHT, Order.FORWARD, "CPU-runnable reference case"),
    2: Workload(2, 4096, 4096, 192, np.float64, Side.RIGHT, Order.FORWARD, "single-GPU wavefront case"),
    3: Workload(3, 65536, 2048, 256, np.float64, Side.RIGHT, Order.FORWARD, "tall, row-sharded 1/2/4/8 GPUs"),
    4: Workload(4, 8192, 8192, 128, np.float32, Side.RIGHT, Order.FORWARD, "fp32 pipe"),
    5: Workload(5, 16384, 16384, 96, np.float64, Side.LEFT, Order.REVERSE, "QR-sweep-like, column-sharded"),
}


def make_workload_inputs(w: Workload, owner_range=None):
    """(A, C, S) host arrays for workload w (A column-major, C/S (len-1) x k F-order).

    ``owner_range=(o0, o1)`` returns only those rows (right side) / columns (left
    side) of A, generated identically to the full matrix (the generator stream is
    produced in full and sliced, so shards are bit-identical to the full input).
    """
    # right-side row shards: the C-order normal stream yields rows in order, so the
    # first o1 rows of it are exactly rows [0, o1) of the full matrix (no need to
    # generate the rest); left-side column shards need the full stream
    rows = w.m
    if owner_range is not None and w.side is Side.RIGHT:
        rows = owner_range[1]
    if w.index in (1, 2, 3):
        rng = np.random.Generator(np.random.Philox(0))
        A = rng.standard_normal((rows, w.n))
        seq = generate_sequence(w.n, w.k, 1)
        C, S = seq.C, seq.S
    elif w.index == 4:
        rng = np.random.Generator(np.random.Philox(0))
        A = rng.uniform(-1.0, 1.0, size=(rows, w.n)).astype(np.float32)
        th = np.random.Generator(np.random.Philox(1)).uniform(0.0, 2.0 * np.pi, size=(w.n - 1, w.k))
        C, S = np.cos(th).astype(np.float32), np.sin(th).astype(np.float32)
    elif w.index == 5:
        rng = np.random.Generator(np.random.Philox(0))
        A = rng.standard_normal((w.m, w.n))
        A = np.triu(A, k=-1)  # upper Hessenberg: zero entries i > j + 1
        th = np.random.Generator(np.random.Philox(1)).uniform(-np.pi / 2, np.pi / 2, size=(w.m - 1, w.k))
        C, S = np.cos(th), np.sin(th)
    else:
        raise ValueError(f"unknown workload {w.index}")
    if owner_range is not None:
        o0, o1 = owner_range
        A = A[:, o0:o1] if w.side is Side.LEFT else A[o0:o1, :]
    return np.asfortranarray(A), np.asfortranarray(C), np.asfortranarray(S)


def shard_range(total: int, world: int, rank: int, align: int = 64):
    """Balanced contiguous [o0, o1) of `total` owners for `rank`, in units of `align`
    (the CTA tile), leftovers to the last populated shard — the reference's
    partition_rows rule (blocking.py:178-202) applied to GPUs."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    units, rem = divmod(total, align)
    base, extra = divmod(units, world)
    lengths = [(base + (1 if i < extra else 0)) * align for i in range(world)]
    last = max([i for i, ln in enumerate(lengths) if ln > 0], default=world - 1)
    lengths[last] += rem
    start = sum(lengths[:rank])
    return start, start + lengths[rank]

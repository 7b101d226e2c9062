"""paper_2412_01852_b200 — B200-native application of plane-rotation sequences.

A from-scratch sm_100a implementation of the hot path of the ``rotseq``
reference package (arXiv 2412.01852): apply k sweeps of (n-1) Givens rotations,
stored as (n-1) x k cosine/sine arrays C and S, to an m x n column-major matrix
in place. Python mirrors the reference's entry points; the arithmetic runs in
hand-written CUDA kernels behind the C-ABI in ``include/rotseq_b200.h``.
"""

from .core import (  # noqa: F401
    Order,
    RotationSequence,
    Side,
    TransformKind,
    check_apply_args,
    flops_applied,
    generate_sequence,
    make_inputs,
    require_colmajor,
)
from .compare import (  # noqa: F401
    EPS,
    EPS32,
    ComparisonReport,
    baseline_tol,
    compare,
    fast_mode_tol,
    norm_preservation_tol,
)
from .apply import (  # noqa: F401
    PackedSequence,
    apply_blocked,
    apply_cuda,
    apply_device,
    apply_dmma,
    dmma_workspace_bytes,
    apply_host,
    apply_naive,
    workspace_bytes,
)
from .workloads import WORKLOADS, Workload, make_workload_inputs, shard_range  # noqa: F401
from .verification import ALGORITHMS, FAULT_ENV, run_variant  # noqa: F401

__version__ = "0.1.0"

"""Tile model of the B200 pipeline kernel: the counterpart of the reference's memory-
operation model (rotseq/model.py:73-108 ``memops_kernel``) and of its cache-driven block
planner (rotseq/blocking.py:115-147 ``choose_block_sizes``).

The reference sizes (n_b, k_b, m_b) so that a panel, its coefficient tiles and a row block
fit L1 / L2 / L3, and counts element traffic per applied transform as

    kernel  total = (2/k_r + 2/n_b + 2/m_r) * X          (model.py:13)

On the GPU the three levels are the register window of a thread (k_r -> K sweeps per
unit, one column enters and one leaves the window per wave of K transforms), the shared-
memory rings and coefficient buffers of a CTA (m_r -> 32*R rows of a warp share one
broadcast coefficient record), and HBM (A crosses it once per chain of ring-linked units).
``memops_window`` restates the formula in those terms; ``issue_cycles`` turns it into
issue / register-file cycles of one SM sub-partition (SMSP), which is what bounds this
FP-pipe-bound kernel; ``choose_tile_shape`` picks (K, R, warps per CTA) the way
``choose_block_sizes`` picks (n_b, k_b, m_b): the largest window that fits the budgets
(registers per thread, shared memory per CTA, instruction-cache footprint of the unrolled
block), then the row count and warp count with the lowest modelled cycles per transform.

The library's compile-time constants (``rs_tile_shape`` in include/rotseq_b200.h) must equal
this model's choice; tests/test_model.py pins both, and the modelled throughput is compared
with the microbenchmarks of tools/microbench.

Hardware constants measured on B200 (tools/microbench):
  * DFMA: one warp instruction per 2 cycles per SMSP, dependent latency 8.2 cycles
    (dfma_lat.cu);
  * an FMA whose three 64-bit operands are distinct vector registers needs 3 register-file
    read cycles, i.e. it issues at 2/3 of the pipe's rate (dfma_operands.cu: 63.7% of the
    pipe; 97.6% with the multiplier in a uniform register or the constant bank, which the
    toolchain only produces for constant-bank data). When G consecutive DFMAs of a warp
    share their multiplier register the operand reuse cache serves it: 79% (G=2), 85%
    (G=4), 88% (G=8) of the pipe (dfma_reuse.cu) = (2G+1)/G read cycles per G instructions.
    ptxas's schedule keeps ~56% of the possible pairs adjacent (SASS .reuse flags: 28% of
    the DFMAs at R=2 of the possible 50%, 40% of 67% at R=3, 50% of 75% at R=4).
"""

from __future__ import annotations

from dataclasses import dataclass, field

__all__ = [
    "SmSpec", "TileShape", "WindowMemOps", "memops_window", "issue_cycles", "register_need",
    "smem_per_warp", "block_code_bytes", "candidate_table", "fill_efficiency", "choose_tile_shape",
    "modelled_tflops", "TARGET_WORKLOADS",
]


@dataclass(frozen=True)
class SmSpec:
    """One B200 SM (sm_100a) as the model sees it."""

    sms: int = 148
    smsp_per_sm: int = 4
    regs_per_sm: int = 65536
    max_regs_per_thread: int = 255
    reg_alloc_unit: int = 8                 # registers per thread are granted in multiples of 8
    smem_optin_bytes: int = 232448          # 227 KB dynamic shared memory per CTA
    icache_budget_bytes: int = 13312        # unrolled block body that still streams from the
    #                                         instruction cache: 12.7 KB bodies run at full
    #                                         speed (body_r.cu R=4), 14.6 KB (K=12 fp64) and
    #                                         22 KB (K=16 fp32, ncu: 62% no_instruction) do not
    clock_ghz: float = 1.965
    fma_issue_cycles: dict = field(default_factory=lambda: {8: 2.0, 4: 1.0})  # per element size
    rf_read_cycles_3op: dict = field(default_factory=lambda: {8: 3.0, 4: 1.5})  # 3 distinct regs
    reuse_pairing: float = 0.56             # share of the possible multiplier reuses ptxas keeps
    fma_latency_cycles: float = 8.2
    min_warps_per_smsp: int = 3             # fewer cannot cover the hand-off waits (measured:
    #                                         8-warp CTAs lose to 12-warp ones at equal R)
    warp_choices: tuple = (8, 12, 16)
    # Window widths considered: a unit covers K consecutive sweeps and a chain runs at the
    # pace of its widest unit (measured), so K must split the sweep counts
    # in use evenly; those are multiples of 8 (every BASELINE configuration: 64 ... 256).
    window_choices: tuple = (2, 4, 8, 16)


@dataclass(frozen=True)
class TileShape:
    """K sweeps per unit window, R rows per thread (32*R rows per warp tile), warps per CTA
    of the register budget it was sized for, ring depth in chunks of K+1 columns."""

    K: int
    R: int
    warps: int
    ring_chunks: int = 2

    @property
    def tile_rows(self) -> int:
        return 32 * self.R


@dataclass(frozen=True)
class WindowMemOps:
    """Element operations per applied transform element at each level (the reference's
    MemOpReport.per_rotation_factor, split by level)."""

    shared: float       # register window <-> shared-memory ring     (reference term 2/k_r)
    coefficient: float  # coefficient words per element              (reference term 2/m_r)
    hbm: float          # A through HBM                              (reference term 2/n_b)

    @property
    def per_rotation_factor(self) -> float:
        return self.shared + self.coefficient + self.hbm


def memops_window(K: int, R: int, k: int, ring_linked_units: int | None = None) -> WindowMemOps:
    """Element traffic of the register-window kernel per applied transform element.

    One column enters and one leaves the window per wave of K transforms (2/K, the
    reference's 2/k_r); a coefficient pair is read once per warp and wave lane and serves the
    32*R rows of the tile (2/(32 R), the reference's 2/m_r); A crosses HBM once per chain of
    ``ring_linked_units`` consecutive units handed over through shared memory (2 / sweeps of
    the chain; a chain that spans all k sweeps reads and writes A exactly once)."""
    if K < 1 or R < 1 or k < 1:
        raise ValueError(f"window parameters must be positive: K={K}, R={R}, k={k}")
    units = -(-k // K)
    linked = units if ring_linked_units is None else max(1, min(units, ring_linked_units))
    return WindowMemOps(shared=2.0 / K, coefficient=2.0 / (32 * R), hbm=2.0 / min(k, linked * K))


# per-form FP instruction count of one transform element and how many of those are FMAs
# with three distinct register operands (scaled: 2 FMA; fast standard: 2 MUL + 2 FMA;
# strict: 4 MUL + 2 ADD; reflector fast: ADD + MUL + 2 FMA)
_FORMS = {"scaled": (2, 2), "fast": (4, 2), "strict": (6, 0), "reflector": (4, 2)}
PROTOCOL_SLOTS_PER_BLOCK = 60  # barrier waits, arrives, coefficient copy, pointer updates


def issue_cycles(K: int, R: int, tsz: int = 8, form: str = "scaled", spec: SmSpec = SmSpec()) -> dict:
    """Modelled SMSP cycles per transform element of one thread row.

    fp: every FP instruction holds the pipe for ``fma_issue_cycles``; an FMA with three
    distinct register operands holds the register file for ``rf_read_cycles_3op`` unless
    the multiplier (shared by the R rows of the thread) comes from the reuse cache, which
    ptxas achieves for ``reuse_pairing`` of the (R-1)/R possible cases.
    smem: one LDS (column in), one STS (column out) and, in the scaled form, one multiply
    by the column scale per K transforms.  coef: one broadcast LDS.128 per transform and
    warp lane, shared by the R rows (fp32 records hold two lanes).  protocol: the per-block
    hand-off work spread over the block's (K+1)*K*R transform elements."""
    n_fp, n_fma3 = _FORMS[form]
    issue = spec.fma_issue_cycles[tsz]
    rf3 = spec.rf_read_cycles_3op[tsz]
    reused = spec.reuse_pairing * (R - 1) / R
    fp = (n_fp - n_fma3) * issue + n_fma3 * (reused * issue + (1.0 - reused) * max(issue, rf3))
    smem = (2.0 + (issue if form == "scaled" else 0.0)) / K
    coef = (0.5 if tsz == 4 and form != "reflector" else 1.0) / R
    protocol = PROTOCOL_SLOTS_PER_BLOCK / float((K + 1) * K * R)
    return {"fp": fp, "smem": smem, "coef": coef, "protocol": protocol, "total": fp + smem + coef + protocol}


def register_need(K: int, R: int, tsz: int = 8, left: bool = False) -> int:
    """Registers per thread: the (K+1) x R window, one column in flight each way, the
    4-deep coefficient queue (16 registers) and the addressing / protocol state of the
    unit loop (~96 registers on the right side, ~112 on the left with its owner-major chunk
    copies). Calibrated on ptxas: the fp64 R=2 right-side kernel needs 168 (24 bytes of
    spills remain), the fp32 one 128 (40 bytes)."""
    w = tsz // 4
    base = 112 if left else 96
    return w * (K + 1) * R + 2 * w * R + 16 + base


SPILL_TOLERANCE_REGS = 8  # a build a few registers short still runs at speed (measured)


def smem_per_warp(K: int, R: int, tsz: int = 8, ring_chunks: int = 2, left: bool = False) -> int:
    """Shared memory per warp: ``ring_chunks`` chunks of (K+1) columns x 32*R rows and two
    coefficient buffers (two blocks each on the right side) of (K+1)*K 16-byte records plus
    the scaled form's column scales; mirrors smem_per_warp in csrc/rotseq_b200.cu."""
    recs = (K + 1) * ((K + 1) // 2 if tsz == 4 else K)
    scale = ((K + 1) * tsz + 15) // 16
    cbuf = (recs + scale) * 16
    return 2 * (1 if left else 2) * cbuf + ring_chunks * (K + 1) * 32 * R * tsz + (ring_chunks + 3) * 8


def block_code_bytes(K: int, R: int, tsz: int = 8, form: str = "scaled") -> int:
    """Size of the fully unrolled interior block: per wave K transforms of R rows, K
    coefficient loads (fp32: K/2), and per row one LDS, one STS and one scale multiply."""
    n_fp, _ = _FORMS[form]
    coef_loads = (K + 1) // 2 if tsz == 4 else K
    per_wave = K * R * n_fp + coef_loads + 3 * R + 4
    return 16 * (K + 1) * per_wave


def _regs_per_thread(warps: int, spec: SmSpec) -> int:
    r = spec.regs_per_sm // (32 * warps)
    r -= r % spec.reg_alloc_unit
    return min(r, spec.max_regs_per_thread)


def candidate_table(tsz: int = 8, left: bool = False, form: str = "scaled", spec: SmSpec = SmSpec(),
                    ring_chunks: int = 2) -> list[dict]:
    """Every (K, R, warps) with its budgets and modelled cycles; ``feasible`` is false
    with the violated budget named in ``why``."""
    rows = []
    for K in spec.window_choices:
        for R in range(1, 5):
            for warps in spec.warp_choices:
                need = register_need(K, R, tsz, left)
                have = _regs_per_thread(warps, spec)
                smem = warps * smem_per_warp(K, R, tsz, ring_chunks, left) + (ring_chunks + 3) * 8
                code = block_code_bytes(K, R, tsz, form)
                why = []
                if need > have + SPILL_TOLERANCE_REGS:
                    why.append(f"registers {need} > {have}")
                if smem > spec.smem_optin_bytes:
                    why.append(f"shared memory {smem} > {spec.smem_optin_bytes}")
                if code > spec.icache_budget_bytes:
                    why.append(f"block body {code} B > {spec.icache_budget_bytes}")
                if warps // spec.smsp_per_sm < spec.min_warps_per_smsp:
                    why.append(f"{warps // spec.smsp_per_sm} warps per SMSP < {spec.min_warps_per_smsp}")
                cyc = issue_cycles(K, R, tsz, form, spec)
                rows.append({"K": K, "R": R, "warps": warps, "registers": need, "register_budget": have,
                             "smem_bytes": smem, "code_bytes": code, "cycles": cyc["total"], "terms": cyc,
                             "feasible": not why, "why": "; ".join(why)})
    return rows


# (owners, sweeps) of the BASELINE configurations each kernel family has to serve: the
# compile-time shape is chosen for the worst of them (configs 2 and 3; 5; 4 and, for the
# fp32 left side, which BASELINE does not exercise, its transpose)
TARGET_WORKLOADS = {
    (8, False): ((4096, 192), (65536, 256)),
    (8, True): ((16384, 96),),
    (4, False): ((8192, 128),),
    (4, True): ((8192, 128),),
}


def fill_efficiency(K: int, R: int, warps: int, owners: int, k: int, spec: SmSpec = SmSpec()) -> float:
    """Share of the chip's warp slots a problem keeps busy with this shape: its units
    (tiles of 32*R owners x ceil(k/K) sweep ranges) run in whole rounds of sms*warps
    slots (the GPU counterpart of the reference's partition_rows balance,
    blocking.py:178-202). Fat tiles leave a mid-sized problem with too few units."""
    units = -(-owners // (32 * R)) * -(-k // K)
    slots = spec.sms * warps
    rounds = -(-units // slots)
    return units / float(rounds * slots)


def choose_tile_shape(tsz: int = 8, left: bool = False, form: str = "scaled", spec: SmSpec = SmSpec(),
                      ring_chunks: int = 2, workloads=None) -> TileShape:
    """The feasible (K, R, warps) with the highest modelled throughput on the worst of the
    target workloads: steady-state cycles per transform element (issue_cycles) divided by
    the share of the chip the workload fills (fill_efficiency). Ties go to the wider
    window (fewer hand-offs per sweep), then to fewer warps (more registers per thread)."""
    workloads = TARGET_WORKLOADS[(tsz, left)] if workloads is None else workloads
    # one tile height per element size: the left side keeps the right side's rows per
    # thread (tile_owners() in the library is a function of the element size only, so
    # shard boundaries and workspace sizes do not depend on the side)
    rows = choose_tile_shape(tsz, False, form, spec, ring_chunks).R if left else None
    best = None
    for c in candidate_table(tsz, left, form, spec, ring_chunks):
        if not c["feasible"] or (rows is not None and c["R"] != rows):
            continue
        fill = min(fill_efficiency(c["K"], c["R"], c["warps"], o, k, spec) for o, k in workloads)
        key = (round(c["cycles"] / fill, 6), -c["K"], c["warps"])
        if best is None or key < best[0]:
            best = (key, c)
    if best is None:
        raise ValueError("no tile shape fits the SM budgets")
    c = best[1]
    return TileShape(K=c["K"], R=c["R"], warps=c["warps"], ring_chunks=ring_chunks)


def modelled_tflops(shape: TileShape, tsz: int = 8, form: str = "scaled", spec: SmSpec = SmSpec(),
                    active_sms: int | None = None) -> float:
    """Counted TFLOP/s (6 flops per transform element) of the steady-state block body on
    ``active_sms`` SMs: 32 lanes per SMSP cycle budget / modelled cycles."""
    sms = spec.sms if active_sms is None else active_sms
    cyc = issue_cycles(shape.K, shape.R, tsz, form, spec)["total"]
    return 6.0 * 32.0 * sms * spec.smsp_per_sm * spec.clock_ghz / cyc / 1e3

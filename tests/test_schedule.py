"""CPU checks of the CUDA kernel's schedule and algebra (no GPU):

* the hand-off protocol (rings, flags, rounds, tail-first CTA order) is deadlock free
  on the BASELINE geometries and on forced small geometries (pipeline_model);
* the block / wave / lane decomposition applies exactly the (n-1)k transforms in a
  dependency-legal order (the reference's assert_naive_equivalent_order,
  conftest.py:26-43);
* a numpy emulation of the register-window slots and the packed coefficient records
  reproduces the oracle bit for bit (kernel_emulator), and the fast-mode scaled records
  reproduce it within the fast-mode tolerance.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import assert_bitwise, assert_naive_equivalent_order
from kernel_emulator import emulate, pack_unit_scaled, unit_partition
from pipeline_model import Geometry, plan, simulate, unit_block_rotations, warp_cap


@pytest.mark.parametrize("owners,length,k,dtype_bytes,refl", [
    (4096, 4096, 192, 8, False),    # config 2
    (512, 512, 64, 8, False),       # config 1
    (8192, 2048, 256, 8, False),    # config 3 per GPU at 8 GPUs
    (8192, 8192, 128, 4, False),    # config 4 (fp32)
    (2048, 16384, 96, 8, False),    # config 5 per GPU at 8 GPUs (columns are owners)
    (4096, 1024, 192, 8, True),     # reflector records (smaller cap)
])
def test_protocol_deadlock_free_on_baseline_geometries(owners, length, k, dtype_bytes, refl):
    g = Geometry(owners=owners, length=length, k=k)
    res = simulate(g, cap=warp_cap(dtype_bytes, refl))
    assert res["plan"]["G"] >= 1


@pytest.mark.parametrize("cap,grid", [(4, 1), (4, 3), (8, 2), (4, 5), (8, 7), (4, None), (16, 148)])
@pytest.mark.parametrize("owners,length,k", [(100, 50, 40), (300, 37, 33), (64, 200, 70), (33, 9, 24),
                                             (700, 20, 100), (129, 300, 8)])
@pytest.mark.parametrize("mode", (1, 2))
def test_protocol_deadlock_free_forced_geometries(cap, grid, owners, length, k, mode):
    """The RS_DEBUG_MAX_WARPS / RS_DEBUG_GRID / RS_PLAN_MODE geometries run on the GPU."""
    simulate(Geometry(owners=owners, length=length, k=k), cap=cap, grid=grid, mode=mode)


def test_plan_balances_sub_partitions():
    """Config 2: every SM sub-partition gets exactly q units of nearly equal width."""
    g = Geometry(owners=4096, length=4096, k=192)
    pl = plan(g, cap=16)
    assert pl["U"] % (4 * pl["G"]) == 0
    from pipeline_model import cta_schedule
    for c in (0, 1, 77, pl["G"] - 1):
        loads = [0, 0, 0, 0]
        for _, w, _, _, (_, _, kb), _, _ in cta_schedule(g, pl, c):
            loads[w % 4] += kb
        assert max(loads) - min(loads) <= 2, loads


@pytest.mark.parametrize("k,ut", [(192, 27), (192, 28), (7, 7), (100, 13), (8, 1)])
def test_unit_partition_covers_sweeps(k, ut):
    parts = unit_partition(k, ut)
    assert parts[0][0] == 0 and sum(kb for _, kb in parts) == k
    assert all(1 <= kb <= 8 for _, kb in parts) or ut * 8 < k
    assert all(parts[i][0] + parts[i][1] == parts[i + 1][0] for i in range(ut - 1))


@pytest.mark.parametrize("length,k,ut", [(2, 1, 1), (3, 5, 1), (9, 8, 1), (10, 8, 2), (17, 9, 2), (40, 24, 4),
                                         (33, 100, 13), (64, 7, 3)])
def test_block_decomposition_is_dependency_legal(length, k, ut):
    g = Geometry(owners=64, length=length, k=k)
    order = []
    # units run in pipeline order; any interleaving that respects the ring protocol
    # keeps unit i+1 behind unit i per column, so the unit-sequential order suffices
    for p0, kb in unit_partition(k, ut):
        for b in range(g.nblk):
            order.extend(unit_block_rotations(g, p0, kb, b))
    assert_naive_equivalent_order(order, length, k)


def test_pipelined_interleaving_is_dependency_legal():
    """The actual interleaving of unit blocks produced by the protocol model."""
    g = Geometry(owners=200, length=60, k=40)
    res = simulate(g, cap=4, grid=4)
    for tile, events in res["order"].items():
        order = [r for p0, kb, b in events for r in unit_block_rotations(g, p0, kb, b)]
        assert_naive_equivalent_order(order, g.length, g.k)


@pytest.mark.parametrize("side", ("right", "left"))
@pytest.mark.parametrize("order", ("forward", "reverse"))
@pytest.mark.parametrize("kind", ("rotation", "reflector"))
def test_kernel_emulator_matches_oracle(oracle_mod, side, order, kind):
    from paper_2412_01852_b200 import generate_sequence, make_inputs

    for (m, n, k, ut) in ((7, 12, 3, 1), (5, 20, 11, 2), (9, 3, 9, 3), (4, 2, 1, 1), (6, 15, 17, 4)):
        A0, seq = make_inputs(m, n, k, 5)
        C, S = seq.C, seq.S
        if side == "left":
            s2 = generate_sequence(m, k, 9)
            C, S = s2.C, s2.S
        ref = A0.copy(order="F")
        oracle_mod.apply_naive(ref, C, S, side=side, order=order, kind=kind)
        assert_bitwise(ref, emulate(A0, C, S, side, order, kind, ut=ut), f"{m}x{n} k={k} {side} {order} {kind}")


@pytest.mark.parametrize("side", ("right", "left"))
@pytest.mark.parametrize("order", ("forward", "reverse"))
@pytest.mark.parametrize("kind", ("rotation", "reflector"))
def test_scaled_form_matches_oracle(oracle_mod, side, order, kind):
    """The fast-mode scaled ("fast Givens") records reproduce the transform within the
    fast-mode tolerance (relative Frobenius <= 10*k*eps)."""
    from paper_2412_01852_b200 import compare, generate_sequence, make_inputs

    for (m, n, k, ut) in ((7, 12, 3, 1), (5, 20, 11, 2), (6, 40, 24, 4), (4, 2, 1, 1)):
        A0, seq = make_inputs(m, n, k, 3)
        C, S = seq.C, seq.S
        if side == "left":
            s2 = generate_sequence(m, k, 4)
            C, S = s2.C, s2.S
        ref = A0.copy(order="F")
        oracle_mod.apply_naive(ref, C, S, side=side, order=order, kind=kind)
        got = emulate(A0, C, S, side, order, kind, ut=ut, scaled=True)
        rep = compare(ref, got, "fast", k=k)
        assert rep.passed, f"{m}x{n} k={k} {side} {order} {kind}: {rep}"


def test_scaled_pack_flags_unsafe_coefficients():
    """c == 0 (a quarter turn) has no scaled form: the pack must report it so the
    kernel falls back to the standard records."""
    C = np.full((5, 3), 0.6)
    S = np.full((5, 3), 0.8)
    assert not pack_unit_scaled(C, S, 6, 0, 3)[2]
    C[2, 1], S[2, 1] = 0.0, 1.0
    assert pack_unit_scaled(C, S, 6, 0, 3)[2]


def test_kernel_emulator_golden(golden):
    for i in (3, 5, 11):
        A = golden[f"c{i}_A"]
        got = emulate(A, golden[f"c{i}_C"], golden[f"c{i}_S"])
        assert_bitwise(golden[f"c{i}_rot_right_fwd"], got)


@pytest.mark.parametrize("owners,length,k,cap,expect", [
    (4096, 4096, 192, 16, dict(G=144, NW=12, U=1728)),     # config 2: equal chains of 27 units (7-8 sweeps)
    (8192, 8192, 128, 16, dict(G=128, NW=16, U=2048)),     # config 4: 1 CTA per chain
    (16384, 16384, 96, 12, dict(G=128, NW=12, U=3072)),    # config 5: 2 rounds, 1 chain each
    (65536, 2048, 256, 16, dict(G=148, NW=16, U=32768)),   # config 3: many rounds keep all SMs
])
def test_aligned_plans_for_baseline_configs(owners, length, k, cap, expect):
    """The planner picks uniform-width, chain-aligned plans for the few-round BASELINE
    configs and keeps every SM for the many-round config 3."""
    g = Geometry(owners=owners, length=length, k=k)
    pl = plan(g, cap=cap)
    assert {key: pl[key] for key in expect} == expect
    if pl["G"] == 128:
        assert pl["t1"] == 0 and k % pl["ua"] == 0  # every unit exactly k/ut sweeps wide


def test_equal_chain_plan_for_config_2():
    """Config 2: the aligned plan (24 units of 8 sweeps, 128 CTAs, chains crossing CTAs) gives
    way to equal chains of 27 units on 144 CTAs; the three 8-sweep units of a chain sit at
    positions 7, 16, 25 — never the head, the tail or a flag hand-off unit of any tile."""
    from pipeline_model import cta_schedule, unit_at
    g = Geometry(owners=4096, length=4096, k=192)
    aligned = plan(g, cap=16, equal_chain=False)
    assert (aligned["G"], aligned["NW"], aligned["U"], aligned["off"]) == (128, 12, 1536, 0)
    pl = plan(g, cap=16)
    assert (pl["G"], pl["NW"], pl["U"], pl["ua"], pl["t1"]) == (144, 12, 1728, 27, 0)
    widths = [unit_at(i, 0, 27, 192, pl["off"])[2] for i in range(27)]
    assert sum(widths) == 192 and [i for i, w in enumerate(widths) if w == 8] == [7, 16, 25]
    for c in range(pl["G"]):
        loads = [0, 0, 0, 0]
        for _, w, _, _, (_, p0, kb), src, dst in cta_schedule(g, pl, c):
            loads[w % 4] += kb
            if kb == 8:  # a wide unit is a plain ring-to-ring stage
                assert (src, dst) == ("ring", "ring")
        assert max(loads) <= 22 and min(loads) >= 21, loads
    # a chain that fits one CTA keeps its aligned plan (config 4: no flag hand-off to add)
    assert plan(Geometry(owners=8192, length=8192, k=128), cap=16)["G"] == 128


def test_equal_chain_plan_protocol_is_deadlock_free():
    res = simulate(Geometry(owners=1024, length=2100, k=192), sms=37, cap=16)
    assert (res["plan"]["G"], res["plan"]["ua"]) == (36, 27)


@pytest.mark.parametrize("owners,length,k,cap", [(16384, 16384, 96, 12), (16384, 2048, 256, 16)])
def test_protocol_deadlock_free_on_multi_round_aligned_plans(owners, length, k, cap):
    """Config 5 on one GPU (2 rounds, one chain per round) and the 4-GPU shard of config 3
    (4 rounds): the aligned plans' ring and flag hand-offs complete in the simulation."""
    res = simulate(Geometry(owners=owners, length=length, k=k), cap=cap)
    assert res["plan"]["G"] == 128

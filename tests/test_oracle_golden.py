"""Pin the CPU oracle to the reference: every function in oracle/ must reproduce the
golden vectors the reference itself produced (tests/golden/make_golden.py), bit for
bit in strict mode. CPU only."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import assert_bitwise, assert_naive_equivalent_order  # noqa: F401

KINDS = ("rot", "refl")
KIND_NAME = {"rot": "rotation", "refl": "reflector"}


def cases(golden):
    return [(i, tuple(int(v) for v in c)) for i, c in enumerate(golden["cases"])]


def test_golden_file_has_all_cases(golden):
    assert len(golden["cases"]) >= 10
    for i, (m, n, k, seed) in cases(golden):
        assert golden[f"c{i}_A"].shape == (m, n)
        assert golden[f"c{i}_C"].shape == (n - 1, k)


@pytest.mark.parametrize("kind", KINDS)
def test_c_oracle_naive_right_forward(golden, oracle_mod, kind):
    for i, (m, n, k, seed) in cases(golden):
        A = golden[f"c{i}_A"].copy(order="F")
        oracle_mod.apply_naive(A, golden[f"c{i}_C"], golden[f"c{i}_S"], kind=KIND_NAME[kind])
        assert_bitwise(golden[f"c{i}_{kind}_right_fwd"], A, f"case {i} {kind}")


@pytest.mark.parametrize("kind", KINDS)
def test_c_oracle_naive_right_reverse(golden, oracle_mod, kind):
    for i, (m, n, k, seed) in cases(golden):
        A = golden[f"c{i}_A"].copy(order="F")
        oracle_mod.apply_naive(A, golden[f"c{i}_C"], golden[f"c{i}_S"], order="reverse", kind=KIND_NAME[kind])
        assert_bitwise(golden[f"c{i}_{kind}_right_rev"], A, f"case {i} {kind} reverse")


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("order", ("fwd", "rev"))
def test_c_oracle_naive_left(golden, oracle_mod, kind, order):
    for i, (m, n, k, seed) in cases(golden):
        if f"c{i}_{kind}_left_{order}" not in golden:
            continue
        A = golden[f"c{i}_A"].copy(order="F")
        oracle_mod.apply_naive(A, golden[f"c{i}_Cl"], golden[f"c{i}_Sl"], side="left",
                               order="reverse" if order == "rev" else "forward", kind=KIND_NAME[kind])
        assert_bitwise(golden[f"c{i}_{kind}_left_{order}"], A, f"case {i} {kind} left {order}")


@pytest.mark.parametrize("kind", KINDS)
def test_numpy_oracle_matches_golden(golden, oracle_mod, kind):
    for i, (m, n, k, seed) in cases(golden):
        if m * n * k > 2_000_000:
            continue
        A = golden[f"c{i}_A"].copy(order="F")
        oracle_mod.numpy_apply_naive(A, golden[f"c{i}_C"], golden[f"c{i}_S"], kind=KIND_NAME[kind])
        assert_bitwise(golden[f"c{i}_{kind}_right_fwd"], A, f"numpy case {i}")
        if f"c{i}_{kind}_left_rev" in golden:
            A = golden[f"c{i}_A"].copy(order="F")
            oracle_mod.numpy_apply_naive(A, golden[f"c{i}_Cl"], golden[f"c{i}_Sl"], side="left", order="reverse",
                                         kind=KIND_NAME[kind])
            assert_bitwise(golden[f"c{i}_{kind}_left_rev"], A, f"numpy left rev case {i}")


@pytest.mark.parametrize("threads", (1, 3))
def test_c_oracle_blocked_kernel_tier_bitwise(golden, oracle_mod, threads):
    """The reference's kernel tier is bit-identical to naive in strict mode
    (SPEC criterion 1); its C restatement must be too, for any thread count."""
    for i, (m, n, k, seed) in cases(golden):
        A = golden[f"c{i}_A"].copy(order="F")
        oracle_mod.apply_blocked(A, golden[f"c{i}_C"], golden[f"c{i}_S"], threads=threads)
        assert_bitwise(golden[f"c{i}_rot_right_fwd"], A, f"blocked case {i}")
        assert_bitwise(golden[f"c{i}_rot_blocked"], A, f"reference blocked case {i}")


def test_c_oracle_blocked_small_plans(golden, oracle_mod):
    """Reference variant plans (verification.py:133-157) also give the naive result."""
    i = 4
    for plan in (dict(n_b=8, k_b=2, m_b=16, m_r=16, k_r=2), dict(n_b=7, k_b=3, m_b=40, m_r=8, k_r=5),
                 dict(n_b=13, k_b=5, m_b=24, m_r=12, k_r=3)):
        A = golden[f"c{i}_A"].copy(order="F")
        oracle_mod.apply_blocked(A, golden[f"c{i}_C"], golden[f"c{i}_S"], plan=plan, threads=2)
        assert_bitwise(golden[f"c{i}_rot_right_fwd"], A, f"plan {plan}")


def test_c_oracle_fast_within_tolerance(golden, oracle_mod):
    from paper_2412_01852_b200 import compare

    for i, (m, n, k, seed) in cases(golden):
        A = golden[f"c{i}_A"].copy(order="F")
        oracle_mod.apply_naive(A, golden[f"c{i}_C"], golden[f"c{i}_S"], fast=True)
        assert compare(golden[f"c{i}_rot_right_fwd"], A, "fast", k=k).passed
        B = golden[f"c{i}_A"].copy(order="F")
        oracle_mod.apply_blocked(B, golden[f"c{i}_C"], golden[f"c{i}_S"], fast=True, threads=2)
        assert compare(golden[f"c{i}_rot_right_fwd"], B, "fast", k=k).passed


def test_fp32_oracle_is_fp64_on_rounded_inputs(golden, oracle_mod):
    for i in range(2):
        got = oracle_mod.upcast_reference(golden[f"f{i}_A"], golden[f"f{i}_C"], golden[f"f{i}_S"])
        assert_bitwise(golden[f"f{i}_rot_right_fwd_f64ref"], got, f"fp32 case {i}")


def test_accumulated_q_chain(golden, oracle_mod):
    Q = oracle_mod.accumulate_q(golden["q_C"], golden["q_S"])
    assert_bitwise(golden["q_Q"], Q)
    A = golden["q_A"].copy(order="F")
    oracle_mod.apply_naive(A, golden["q_C"], golden["q_S"])
    assert np.linalg.norm(A - golden["q_AQ"]) / np.linalg.norm(golden["q_AQ"]) <= 1e-12


def test_non_orthonormal_sequence(golden, oracle_mod):
    A = golden["nonorth_A"].copy(order="F")
    oracle_mod.apply_naive(A, golden["nonorth_C"], golden["nonorth_S"])
    assert_bitwise(golden["nonorth_out"], A)


def test_known_answers(oracle_mod):
    """test_rot_ops.py:12-35 / test_variants.py:36-41 of the reference."""
    A = np.asfortranarray([[1.0, 2.0]])
    oracle_mod.apply_naive(A, [[0.6]], [[0.8]])
    assert A[0, 0] == 0.6 * 1.0 + 0.8 * 2.0 and A[0, 1] == 0.6 * 2.0 - 0.8 * 1.0
    A = np.asfortranarray([[1.0, 2.0]])
    oracle_mod.apply_naive(A, [[0.0]], [[1.0]])
    assert A[0, 0] == 2.0 and A[0, 1] == -1.0
    A = np.asfortranarray([[3.0, 4.0]])
    oracle_mod.apply_naive(A, [[1.0]], [[0.0]], kind="reflector")
    assert A[0, 0] == 3.0 and A[0, 1] == -4.0
    A = np.asfortranarray([[3.0, 4.0]])
    oracle_mod.apply_naive(A, [[0.0]], [[1.0]], kind="reflector")
    assert A[0, 0] == 4.0 and A[0, 1] == 3.0


def test_explicit_rotation_products(oracle_mod):
    """Dense G-product oracle (test_variants.py:44-59): G[j,j]=c, G[j,j+1]=-s,
    G[j+1,j]=s, G[j+1,j+1]=c, A <- A @ G."""
    from paper_2412_01852_b200 import make_inputs

    A0, seq = make_inputs(2, 3, 2, 0)
    expect = A0.copy()
    for p in range(2):
        for j in range(2):
            G = np.eye(3)
            c, s = seq.C[j, p], seq.S[j, p]
            G[j, j], G[j, j + 1], G[j + 1, j], G[j + 1, j + 1] = c, -s, s, c
            expect = expect @ G
    got = A0.copy(order="F")
    oracle_mod.apply_naive(got, seq.C, seq.S)
    assert np.allclose(got, expect, rtol=1e-13)


def test_partition_rows_matches_reference_rule(oracle_mod):
    """partition_rows (blocking.py:178-202) invariants."""
    for m, threads, m_r in ((1000, 3, 128), (5, 4, 2), (128, 1, 128), (3, 5, 4), (4096, 16, 128)):
        rs = oracle_mod.partition_rows(m, threads, m_r)
        assert rs[0][0] == 0 and rs[-1][1] == m
        for (a0, a1), (b0, b1) in zip(rs, rs[1:]):
            assert a1 == b0
        lens = [b - a for a, b in rs]
        units = [ln // m_r for ln in lens]
        assert max(units) - min(units) <= 1 + (m % m_r > 0)

"""Host-side mirror of the reference API: validation messages, data model,
generators, comparison profiles, dispatch registry. CPU only (no kernel runs)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import assert_bitwise, make_matrix
from paper_2412_01852_b200 import (
    ALGORITHMS,
    Order,
    RotationSequence,
    Side,
    TransformKind,
    WORKLOADS,
    apply_cuda,
    baseline_tol,
    compare,
    fast_mode_tol,
    flops_applied,
    generate_sequence,
    make_inputs,
    make_workload_inputs,
    run_variant,
    shard_range,
)


def test_generate_sequence_matches_reference(golden):
    g = generate_sequence(10, 4, 1)
    assert_bitwise(golden["gen_C"], g.C)
    assert_bitwise(golden["gen_S"], g.S)


def test_make_inputs_matches_reference(golden):
    for i, c in enumerate(golden["cases"]):
        m, n, k, seed = (int(v) for v in c)
        A, seq = make_inputs(m, n, k, seed)
        assert_bitwise(golden[f"c{i}_A"], A)
        assert_bitwise(golden[f"c{i}_C"], seq.C)
        assert_bitwise(golden[f"c{i}_S"], seq.S)
        assert A.flags.f_contiguous


def test_sequence_validation():
    with pytest.raises(ValueError, match="share a 2-D shape"):
        RotationSequence.from_arrays(np.ones((3, 2)), np.ones((2, 2)))
    with pytest.raises(ValueError, match="at least one"):
        RotationSequence.from_arrays(np.ones((0, 2)), np.ones((0, 2)))
    with pytest.raises(ValueError, match="deviates"):
        RotationSequence.from_arrays([[0.9]], [[0.9]])
    seq = RotationSequence.from_arrays([[0.9]], [[0.9]], check_orthonormal=False)
    assert not seq.orthonormal and seq.n_cols == 2
    with pytest.raises(ValueError, match="n >= 2"):
        generate_sequence(1, 3, 0)
    with pytest.raises(ValueError, match="k >= 1"):
        generate_sequence(4, 0, 0)


def test_apply_validation_messages_before_any_gpu_work():
    """Same message substrings the reference tests match (test_variants.py:62-73,
    test_rot_ops.py:38-45); raised on the host, so this runs without a GPU."""
    A, seq = make_inputs(4, 6, 2, 0)
    with pytest.raises(ValueError, match="acts on"):
        apply_cuda(make_matrix(4, 7), seq)
    with pytest.raises(ValueError, match="column-major"):
        apply_cuda(np.ascontiguousarray(make_matrix(4, 6)), seq)
    with pytest.raises(ValueError, match="float64"):
        apply_cuda(np.asfortranarray(np.zeros((4, 6), dtype=np.int32)), seq)
    with pytest.raises(ValueError, match="2-D"):
        apply_cuda(np.zeros(6), seq)
    with pytest.raises(ValueError, match="at least 2 columns"):
        apply_cuda(np.asfortranarray(np.zeros((4, 1))), generate_sequence(2, 1, 0))
    with pytest.raises(ValueError, match="acts on 6 rows"):
        apply_cuda(make_matrix(5, 6), seq, side="left")
    with pytest.raises(ValueError, match="side"):
        apply_cuda(A, seq, side="middle")
    with pytest.raises(ValueError, match="kind"):
        apply_cuda(A, seq, kind="shear")


def test_zero_rows_is_noop_without_gpu():
    A, seq = make_inputs(0, 6, 3, 0)
    apply_cuda(A, seq)  # m = 0: nothing to do (blocking.py:446-447)


def test_run_variant_registry():
    assert "cuda" in ALGORITHMS and "cuda-naive" in ALGORITHMS
    A, seq = make_inputs(3, 4, 1, 0)
    with pytest.raises(ValueError, match="unknown algorithm"):
        run_variant("kernel", A, seq)


def test_compare_profiles():
    X = make_matrix(8, 9)
    rep = compare(X, X.copy(), "strict")
    assert rep.passed and rep.bitwise_equal
    Y = X.copy()
    Y[0, 0] = np.nextafter(Y[0, 0], np.inf)
    assert not compare(X, Y, "strict").passed
    assert compare(X, Y, "fast", k=3).passed
    assert compare(X, Y, "baseline", k=3).passed
    Z = X * (1 + 1e-6)
    assert not compare(X, Z, "baseline", k=3).passed
    assert fast_mode_tol(4) == 64 * np.finfo(np.float64).eps
    assert baseline_tol(192) == pytest.approx(10 * 192 * 2.220446049250313e-16)
    assert baseline_tol(128, np.float32) == pytest.approx(10 * 128 * 1.1920929e-07)
    with pytest.raises(ValueError, match="profile"):
        compare(X, X, "loose")
    with pytest.raises(ValueError, match="shape mismatch"):
        compare(X, X[:3])


def test_flops_metric():
    """6*m*(n-1)*k (model.py:123-126); left side 6*n*(m-1)*k."""
    assert flops_applied(4096, 4096, 192) == 6.0 * 4096 * 4095 * 192
    assert flops_applied(16384, 16384, 96, Side.LEFT) == 6.0 * 16384 * 16383 * 96
    assert WORKLOADS[2].flops == pytest.approx(19.32e9, rel=1e-3)
    assert WORKLOADS[3].flops == pytest.approx(206.06e9, rel=1e-3)


def test_workload_definitions():
    w1 = WORKLOADS[1]
    A, C, S = make_workload_inputs(w1)
    A2, seq = make_inputs(512, 512, 64, 0)
    assert_bitwise(A2, A)
    assert_bitwise(seq.C, C)
    w5 = WORKLOADS[5]
    assert w5.side is Side.LEFT and w5.order is Order.REVERSE and w5.length == 16384


def test_workload_shards_are_slices_of_the_full_input():
    w = WORKLOADS[1]
    A, C, S = make_workload_inputs(w)
    for world in (2, 3):
        parts = [make_workload_inputs(w, owner_range=shard_range(w.owners, world, r))[0] for r in range(world)]
        assert_bitwise(A, np.asfortranarray(np.concatenate(parts, axis=0)))


@pytest.mark.parametrize("total,world", [(65536, 8), (4096, 3), (100, 4), (63, 2), (5000, 7)])
def test_shard_range_partitions(total, world):
    rs = [shard_range(total, world, r, align=64) for r in range(world)]
    assert rs[0][0] == 0 and rs[-1][1] == total
    for (a0, a1), (b0, b1) in zip(rs, rs[1:]):
        assert a1 == b0
    populated = [i for i, (a0, a1) in enumerate(rs) if a1 > a0]
    for i, (a0, a1) in enumerate(rs):
        if i != populated[-1]:
            assert (a1 - a0) % 64 == 0  # leftovers below one tile go to the last populated shard


def test_enums_accept_strings():
    A, seq = make_inputs(0, 4, 1, 0)
    apply_cuda(A, seq, kind="reflector", side="right", order="reverse")
    assert TransformKind("rotation") is TransformKind.ROTATION


def test_cli_argument_errors_exit_2(capsys):
    """rotbench-compatible CLI: a ValueError (here: run without --n) exits 2 before any
    GPU work, as the reference CLI does (cli.py:372-374); argparse rejects bad choices."""
    from paper_2412_01852_b200 import cli

    assert cli.main(["run", "--algo", "cuda"]) == 2
    assert "needs --n" in capsys.readouterr().err
    with pytest.raises(SystemExit):
        cli.main(["run", "--algo", "kernel", "--n", "8"])

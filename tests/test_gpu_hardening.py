"""GPU parity where round 1 was thin (all through the C-ABI, checked against the oracle).

* fast (scaled "fast Givens") mode under adversarial coefficients: tiny |c| (1e-8 ..
  1e-15), chains of small c across a unit's sweeps up to and past the scaled form's
  range gate, theta -> +-pi/2 (config 5's law), exact swaps (c = 0) and the reference's
  non-orthonormal sequences (conftest.py:46-50 of the reference) — all within BASELINE's
  10*k*eps of the strict oracle, with the per-unit form split reported by rs_packed_form;
* a caller stream different from the current one, with C/S that need a device copy,
  a dtype conversion and compaction (the library must not read them early);
* the multi-GPU code path under torchrun with the NCCL backend (world size 1 — this run
  has one GPU): distributed.apply_sharded with its default CUDA apply, and bench.py's
  torchrun branch (NCCL broadcast inside the timed step);
* the harness: ``cli verify`` passes, and fails (exit 1) with ``--perturb-kernel``
  (reference: cli.py:243-278, tests/test_cli.py:137-144).
"""

from __future__ import annotations

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, assert_bitwise

pytestmark = pytest.mark.gpu

EPS = float(np.finfo(np.float64).eps)


def _gpu_apply(A0, C, S, fast, side="right", order="forward", kind="rotation"):
    import torch

    from paper_2412_01852_b200 import PackedSequence

    dA = torch.from_numpy(A0.copy(order="F")).cuda()
    ps = PackedSequence((torch.from_numpy(C).cuda(), torch.from_numpy(S).cuda()), dA.shape, kind=kind, side=side,
                        order=order, fast_only=fast)
    form = ps.form() if fast else None
    ps.apply(dA, fast=fast)
    return dA.cpu().numpy(), form


def _check_fast(oracle_mod, A0, C, S, side="right", order="forward", kind="rotation", tol_k=None):
    from paper_2412_01852_b200 import compare

    ref = A0.copy(order="F")
    oracle_mod.apply_naive(ref, C, S, side=side, order=order, kind=kind)
    got, form = _gpu_apply(A0, C, S, True, side, order, kind)
    k = C.shape[1]
    rep = compare(ref, got, "baseline", k=tol_k or k)
    assert rep.passed, f"fast result outside 10*k*eps of the strict oracle: {rep} (form {form})"
    # the strict path stays bit-identical on the same adversarial inputs
    strict, _ = _gpu_apply(A0, C, S, False, side, order, kind)
    assert_bitwise(ref, strict, "strict on adversarial coefficients")
    return form, rep


def _theta_cs(theta):
    return np.asfortranarray(np.cos(theta)), np.asfortranarray(np.sin(theta))


@pytest.mark.parametrize("cmag", [1e-8, 1e-12, 1e-15])
def test_fast_tiny_cosines(cuda, oracle_mod, cmag):
    """A tenth of the rotations have |c| = cmag (s = +-sqrt(1 - c^2)): taus ~ 1/cmag."""
    from paper_2412_01852_b200 import make_inputs

    m, n, k = 200, 300, 40
    A0, seq = make_inputs(m, n, k, 5)
    rng = np.random.Generator(np.random.Philox(77))
    C, S = seq.C.copy(order="F"), seq.S.copy(order="F")
    mask = rng.random(C.shape) < 0.1
    sign_c = np.where(rng.random(C.shape) < 0.5, -1.0, 1.0)
    sign_s = np.where(rng.random(C.shape) < 0.5, -1.0, 1.0)
    C[mask] = sign_c[mask] * cmag
    S[mask] = sign_s[mask] * np.sqrt(1.0 - cmag * cmag)
    form, _ = _check_fast(oracle_mod, A0, C, S)
    # a column's scale multiplies up to 16 cosines per unit: at this density |c| = 1e-15
    # pushes most units past the 2^-256 gate (they fall back per unit), 1e-8 and 1e-12
    # almost never do
    if cmag >= 1e-12:
        assert form[0] > 0, f"tiny but in-range cosines should keep the scaled form ({form})"


@pytest.mark.parametrize("cmag,expect_fallback", [(1e-8, False), (1e-12, True)])
def test_fast_small_cosine_chains(cuda, oracle_mod, cmag, expect_fallback):
    """Columns whose rotations have small |c| in every sweep of a unit: the column
    scales multiply up to cmag^8 (1e-64 stays inside the 2^-256 gate, 1e-96 does not),
    so the gate is approached and crossed; crossing it falls back per unit."""
    from paper_2412_01852_b200 import make_inputs

    m, n, k = 150, 120, 32
    A0, seq = make_inputs(m, n, k, 6)
    C, S = seq.C.copy(order="F"), seq.S.copy(order="F")
    for j in (10, 57, 100):
        C[j, :] = cmag * np.where(np.arange(k) % 2 == 0, 1.0, -1.0)
        S[j, :] = np.sqrt(1.0 - cmag * cmag)
    form, _ = _check_fast(oracle_mod, A0, C, S)
    scaled, total = form
    if expect_fallback:
        assert scaled < total, f"chains of |c| = {cmag} should leave the scaled range ({form})"
    else:
        assert scaled == total, f"chains of |c| = {cmag} stay in range ({form})"


def test_fast_theta_near_half_pi_config5_law(cuda, oracle_mod):
    """Config 5's law (theta uniform on [-pi/2, pi/2]) concentrated near +-pi/2, left
    side, reverse order, upper-Hessenberg A."""
    m, n, k = 260, 140, 24
    rng = np.random.Generator(np.random.Philox(0))
    A0 = np.asfortranarray(np.triu(rng.standard_normal((m, n)), k=-1))
    th = np.random.Generator(np.random.Philox(1)).uniform(-np.pi / 2, np.pi / 2, size=(m - 1, k))
    near = np.random.Generator(np.random.Philox(2)).random(th.shape) < 0.3
    th[near] = np.sign(th[near]) * (np.pi / 2 - 10.0 ** -np.random.Generator(np.random.Philox(3)).uniform(
        6, 15, size=near.sum()))
    C, S = _theta_cs(th)
    _check_fast(oracle_mod, A0, C, S, side="left", order="reverse")


@pytest.mark.parametrize("kind", ["rotation", "reflector"])
def test_fast_exact_swaps_fall_back_per_unit(cuda, oracle_mod, kind):
    """c = 0 (an exact swap) is outside the scaled form: only the units holding it run
    the standard form (rs_packed_form), the result is still within 10*k*eps."""
    from paper_2412_01852_b200 import make_inputs

    m, n, k = 256, 400, 64
    A0, seq = make_inputs(m, n, k, 8)
    C, S = seq.C.copy(order="F"), seq.S.copy(order="F")
    C[123, 5] = 0.0
    S[123, 5] = 1.0
    form, _ = _check_fast(oracle_mod, A0, C, S, kind=kind)
    scaled, total = form
    assert 0 < scaled < total, f"one swap must not drop the whole call to the standard form ({form})"
    form_clean, _ = _check_fast(oracle_mod, A0, seq.C, seq.S, kind=kind)
    assert form_clean[0] == form_clean[1]


def test_fast_non_orthonormal(cuda, oracle_mod):
    """The reference's non-orthonormal sequences (C, S ~ U(-1.2, 1.2)) in fast mode."""
    from paper_2412_01852_b200 import make_inputs

    for (m, n, k, seed) in ((64, 48, 3, 0), (100, 70, 6, 1)):
        A0, _ = make_inputs(m, n, k, seed)
        rng = np.random.Generator(np.random.Philox(seed))
        C = np.asfortranarray(rng.uniform(-1.2, 1.2, size=(n - 1, k)))
        S = np.asfortranarray(rng.uniform(-1.2, 1.2, size=(n - 1, k)))
        _check_fast(oracle_mod, A0, C, S)


def test_side_stream_with_converted_cs(cuda, oracle_mod):
    """A caller stream other than the current one, and C/S given as row-major fp32 host
    arrays (device copy + cast + compaction on the current stream first)."""
    import torch

    from paper_2412_01852_b200 import apply_device, make_inputs

    m, n, k = 300, 257, 17
    A0, seq = make_inputs(m, n, k, 4)
    C32 = np.ascontiguousarray(seq.C.astype(np.float32))
    S32 = np.ascontiguousarray(seq.S.astype(np.float32))
    ref = A0.copy(order="F")
    oracle_mod.apply_naive(ref, C32.astype(np.float64), S32.astype(np.float64))
    side = torch.cuda.Stream()
    for _ in range(3):
        dA = torch.from_numpy(A0.copy(order="F")).cuda()
        torch.cuda._sleep(2_000_000)  # keep the current stream busy: an unordered read would race
        Ct = torch.from_numpy(C32).cuda()  # row-major fp32: cast + compaction inside apply_device
        St = torch.from_numpy(S32).cuda()
        apply_device(dA, (Ct, St), fast=False, stream=side)
        del Ct, St  # freed early: record_stream must keep the temporaries alive
        side.synchronize()
        assert_bitwise(ref, dA.cpu().numpy(), "side stream")
    # raw cudaStream_t handle
    dA = torch.from_numpy(A0.copy(order="F")).cuda()
    apply_device(dA, (torch.from_numpy(C32).cuda(), torch.from_numpy(S32).cuda()), fast=False,
                 stream=side.cuda_stream)
    side.synchronize()
    assert_bitwise(ref, dA.cpu().numpy(), "raw stream handle")


def _torchrun(args, timeout=600):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + os.getpid() % 1000), *args]
    return subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout)


@pytest.mark.parametrize("case", [
    (1000, 300, 20, "right", "forward", "rotation", "strict"),
    (200, 500, 12, "left", "reverse", "reflector", "strict"),
    (777, 130, 33, "right", "forward", "rotation", "fast"),
])
def test_torchrun_nccl_apply_sharded(cuda, oracle_mod, tmp_path, case):
    """distributed.apply_sharded, default CUDA apply, NCCL broadcast, under torchrun."""
    from paper_2412_01852_b200 import compare, generate_sequence, make_inputs

    m, n, k, side, order, kind, arith = case
    proc = _torchrun([os.path.join(ROOT, "tests", "nccl_apply_worker.py"), str(tmp_path), str(m), str(n), str(k),
                      side, order, kind, arith])
    assert proc.returncode == 0, proc.stderr[-3000:]
    A, seq = make_inputs(m, n, k, 21)
    if side == "left":
        seq = generate_sequence(m, k, 22)
    ref = A.copy(order="F")
    oracle_mod.apply_naive(ref, seq.C, seq.S, side=side, order=order, kind=kind)
    o0, o1 = np.load(tmp_path / "range0.npy")
    got = np.load(tmp_path / "rank0.npy")
    ref_part = ref[:, o0:o1] if side == "left" else ref[o0:o1, :]
    if arith == "strict":
        assert_bitwise(ref_part, got, "apply_sharded (NCCL, world 1)")
    else:
        rep = compare(ref_part, got, "baseline", k=k)
        assert rep.passed, str(rep)


def test_torchrun_bench_branch(cuda, tmp_path):
    """bench.py under torchrun: NCCL group, C/S broadcast timed inside the step, the
    GPU-count-invariant strict checksum, one JSON line."""
    proc = _torchrun([os.path.join(ROOT, "bench.py"), "--config", "1", "--steps", "3", "--warmup", "3",
                      "--no-e2e", "--no-cpu-baseline"])
    assert proc.returncode == 0, proc.stderr[-3000:]
    lines = [ln for ln in proc.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, proc.stdout
    line = json.loads(lines[0])
    assert line["value"] > 0 and line["gpu_launches"] >= 6
    assert line["phase_ms"]["broadcast"] > 0.0
    # the same checksum without torchrun (no NCCL): identical
    proc2 = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "1", "--steps", "3",
                            "--warmup", "3", "--no-e2e", "--no-cpu-baseline"], cwd=ROOT, capture_output=True,
                           text=True, timeout=600)
    assert proc2.returncode == 0, proc2.stderr[-3000:]
    line2 = json.loads([ln for ln in proc2.stdout.splitlines() if ln.startswith("{")][0])
    assert line2["checksum"] == line["checksum"]


def test_cli_verify_and_fault_injection(cuda, capsys):
    from paper_2412_01852_b200 import cli

    assert cli.main(["verify", "--quick", "--kind", "rotation"]) == 0
    out = capsys.readouterr().out
    assert "cases passed" in out
    assert cli.main(["verify", "--quick", "--kind", "rotation", "--perturb-kernel"]) == 1
    err = capsys.readouterr().err
    assert "FIRST FAILURE cuda" in err
    assert os.environ.get("ROTSEQ_PERTURB_KERNEL") is None  # restored


@pytest.mark.parametrize("kind", ["rotation", "reflector"])
@pytest.mark.parametrize("order", ["forward", "reverse"])
def test_dmma_variant_matches_oracle(cuda, oracle_mod, kind, order):
    """The FP64 tensor-core variant (rs_apply_dmma_f64) against the strict oracle at
    BASELINE's 10*k*eps: partial row tiles, partial passes (k not a multiple of 32),
    windows clipped at both ends, odd lda views."""
    import torch

    from paper_2412_01852_b200 import apply_dmma, compare, make_inputs

    for (m, n, k) in ((64, 64, 32), (100, 70, 40), (33, 300, 7), (257, 129, 65), (8, 2, 3)):
        A0, seq = make_inputs(m, n, k, 13)
        ref = A0.copy(order="F")
        oracle_mod.apply_naive(ref, seq.C, seq.S, order=order, kind=kind)
        got = A0.copy(order="F")
        apply_dmma(got, seq, kind=kind, order=order)
        rep = compare(ref, got, "baseline", k=k)
        assert rep.passed, f"{m}x{n} k={k}: {rep}"
        # a row-block view with odd lda on the device
        big = torch.zeros((n, m + 3), dtype=torch.float64, device="cuda").t()
        view = big[1:m + 1, :]
        view.copy_(torch.from_numpy(A0))
        apply_dmma(view, seq, kind=kind, order=order)
        rep = compare(ref, view.cpu().numpy(), "baseline", k=k)
        assert rep.passed, f"view {m}x{n} k={k}: {rep}"

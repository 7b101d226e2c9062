"""GPU parity of the CUDA path (through the C-ABI) against the reference's golden
vectors and the pinned CPU oracle. Bit-exact in strict mode; fast mode within the
reference's fast profile (16*k*eps) and BASELINE's 10*k*eps."""

from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import assert_bitwise, make_matrix

pytestmark = pytest.mark.gpu

KIND_NAME = {"rot": "rotation", "refl": "reflector"}


def _gpu(A, C, S, **kw):
    from paper_2412_01852_b200 import apply_cuda

    got = np.array(A, order="F", copy=True)
    apply_cuda(got, (C, S), **kw)
    return got


@pytest.mark.parametrize("algo", ("pipeline", "naive"))
@pytest.mark.parametrize("kind", ("rot", "refl"))
def test_golden_vectors_bitwise(cuda, golden, algo, kind):
    """Direct pin to the reference: outputs it produced itself (make_golden.py)."""
    for i, c in enumerate(golden["cases"]):
        A, C, S = golden[f"c{i}_A"], golden[f"c{i}_C"], golden[f"c{i}_S"]
        for order, tag in (("forward", "fwd"), ("reverse", "rev")):
            got = _gpu(A, C, S, kind=KIND_NAME[kind], order=order, algo=algo)
            assert_bitwise(golden[f"c{i}_{kind}_right_{tag}"], got, f"case {i} right {order}")
            key = f"c{i}_{kind}_left_{tag}"
            if key in golden:
                got = _gpu(A, golden[f"c{i}_Cl"], golden[f"c{i}_Sl"], kind=KIND_NAME[kind], order=order,
                           side="left", algo=algo)
                assert_bitwise(golden[key], got, f"case {i} left {order}")


def test_golden_non_orthonormal(cuda, golden):
    got = _gpu(golden["nonorth_A"], golden["nonorth_C"], golden["nonorth_S"])
    assert_bitwise(golden["nonorth_out"], got)


def test_reference_criterion1_grid(cuda, oracle_mod):
    """The reference's full bitwise grid (verification.py:161-195): m in 2..257,
    n in 4..256, k <= 12, both kinds, strict, against the plain loop."""
    from paper_2412_01852_b200 import make_inputs
    from paper_2412_01852_b200.verification import case_grid

    n_cases = 0
    for m, n, k in case_grid(quick=False):
        A0, seq = make_inputs(m, n, k, 7)
        for kind in ("rotation", "reflector"):
            ref = A0.copy(order="F")
            oracle_mod.apply_naive(ref, seq.C, seq.S, kind=kind)
            assert_bitwise(ref, _gpu(A0, seq.C, seq.S, kind=kind), f"m={m} n={n} k={k} {kind}")
            n_cases += 1
    assert n_cases == 684  # 342 (m, n, k) cases x 2 kinds, as in the reference grid


SIDES_ORDERS = [(s, o) for s in ("right", "left") for o in ("forward", "reverse")]


SHAPES = [(1, 2, 1), (2, 2, 3), (3, 9, 3), (63, 65, 8), (64, 64, 16), (65, 40, 17), (200, 31, 50),
          (33, 300, 9), (130, 130, 100), (7, 1000, 24)]


@pytest.mark.parametrize("side,order", SIDES_ORDERS)
@pytest.mark.parametrize("kind", ("rotation", "reflector"))
@pytest.mark.parametrize("m,n,k", SHAPES)
def test_all_variants_bitwise(cuda, oracle_mod, side, order, kind, m, n, k):
    from paper_2412_01852_b200 import generate_sequence, make_inputs

    if side == "left" and m < 2:
        m, n = n, m + 1  # the left side rotates rows: needs m >= 2 (swap the degenerate shape)
    A0, seq = make_inputs(m, n, k, 11)
    if side == "left":
        seq = generate_sequence(m, k, 12)
    ref = A0.copy(order="F")
    oracle_mod.apply_naive(ref, seq.C, seq.S, side=side, order=order, kind=kind)
    assert_bitwise(ref, _gpu(A0, seq.C, seq.S, side=side, order=order, kind=kind))
    assert_bitwise(ref, _gpu(A0, seq.C, seq.S, side=side, order=order, kind=kind, algo="naive"))


@pytest.mark.parametrize("max_warps,grid", [("1", "1"), ("2", "3"), ("3", "2"), ("4", "5"), ("5", "7"), ("2", "")])
def test_forced_multi_round_multi_cta(cuda, oracle_mod, monkeypatch, max_warps, grid):
    """Rings, progress flags, rounds and the tail-first CTA order on small problems."""
    from paper_2412_01852_b200 import generate_sequence, make_inputs

    monkeypatch.setenv("RS_DEBUG_MAX_WARPS", max_warps)
    if grid:
        monkeypatch.setenv("RS_DEBUG_GRID", grid)
    for (m, n, k, side, order, kind) in [(100, 50, 40, "right", "forward", "rotation"),
                                         (300, 37, 33, "right", "reverse", "reflector"),
                                         (64, 200, 70, "right", "forward", "rotation"),
                                         (33, 9, 24, "right", "forward", "reflector"),
                                         (90, 60, 41, "left", "reverse", "reflector"),
                                         (129, 130, 65, "left", "forward", "rotation")]:
        A0, seq = make_inputs(m, n, k, 2)
        if side == "left":
            seq = generate_sequence(m, k, 3)
        ref = A0.copy(order="F")
        oracle_mod.apply_naive(ref, seq.C, seq.S, side=side, order=order, kind=kind)
        assert_bitwise(ref, _gpu(A0, seq.C, seq.S, side=side, order=order, kind=kind),
                       f"{m}x{n} k={k} {side} {order} {kind}")


@pytest.mark.parametrize("kind", ("rotation", "reflector"))
def test_fast_mode_tolerances(cuda, oracle_mod, kind):
    from paper_2412_01852_b200 import compare, make_inputs

    for (m, n, k) in ((40, 48, 6), (300, 500, 64), (1000, 257, 100)):
        A0, seq = make_inputs(m, n, k, 1)
        ref = A0.copy(order="F")
        oracle_mod.apply_naive(ref, seq.C, seq.S, kind=kind)
        got = _gpu(A0, seq.C, seq.S, kind=kind, fast=True)
        assert compare(ref, got, "fast", k=k).passed
        assert compare(ref, got, "baseline", k=k).passed


@pytest.mark.parametrize("side,order", SIDES_ORDERS)
@pytest.mark.parametrize("kind", ("rotation", "reflector"))
def test_fast_mode_scaled_and_standard_forms(cuda, oracle_mod, monkeypatch, side, order, kind):
    """fp64 fast mode runs the scaled ("fast Givens") records; RS_NO_SCALED=1 forces the
    standard 2 MUL + 2 FMA form. Both within 10*k*eps of the strict oracle."""
    from paper_2412_01852_b200 import compare, generate_sequence, make_inputs

    for (m, n, k) in ((70, 90, 17), (130, 600, 40)):
        A0, seq = make_inputs(m, n, k, 2)
        if side == "left":
            seq = generate_sequence(m, k, 5)
        ref = A0.copy(order="F")
        oracle_mod.apply_naive(ref, seq.C, seq.S, side=side, order=order, kind=kind)
        for flag in ("0", "1"):
            monkeypatch.setenv("RS_NO_SCALED", flag)
            got = _gpu(A0, seq.C, seq.S, side=side, order=order, kind=kind, fast=True)
            rep = compare(ref, got, "baseline", k=k)
            assert rep.passed, f"RS_NO_SCALED={flag} {m}x{n} k={k} {side} {order} {kind}: {rep}"


@pytest.mark.parametrize("kind", ("rotation", "reflector"))
def test_fast_mode_unsafe_coefficients_fall_back(cuda, oracle_mod, kind):
    """Quarter turns (c == 0) have no scaled form: the pack flags them and the kernel
    runs the standard records, still within tolerance (and exact for c=0, s=1 swaps)."""
    from paper_2412_01852_b200 import compare, make_inputs

    m, n, k = 200, 300, 24
    A0, seq = make_inputs(m, n, k, 4)
    C, S = seq.C.copy(), seq.S.copy()
    C[::7, ::3], S[::7, ::3] = 0.0, 1.0
    ref = A0.copy(order="F")
    oracle_mod.apply_naive(ref, C, S, kind=kind)
    got = _gpu(A0, C, S, kind=kind, fast=True)
    rep = compare(ref, got, "baseline", k=k)
    assert rep.passed and np.isfinite(got).all(), rep


def test_fp32_strict_bitwise_vs_numpy_fp32_oracle(cuda, oracle_mod):
    for (m, n, k, side, order) in ((65, 33, 12, "right", "forward"), (100, 70, 17, "left", "reverse"),
                                   (31, 200, 40, "right", "reverse")):
        rng = np.random.Generator(np.random.Philox(0))
        A = np.asfortranarray(rng.uniform(-1, 1, (m, n)).astype(np.float32))
        length = m if side == "left" else n
        th = np.random.Generator(np.random.Philox(1)).uniform(0, 2 * np.pi, (length - 1, k))
        C, S = np.cos(th).astype(np.float32), np.sin(th).astype(np.float32)
        ref = A.copy(order="F")
        oracle_mod.numpy_apply_naive(ref, C, S, side=side, order=order)
        assert_bitwise(ref, _gpu(A, C, S, side=side, order=order), f"fp32 {side} {order}")


def test_fp32_fast_vs_fp64_reference(cuda, golden, oracle_mod):
    """BASELINE config-4 rule: the reference in fp64 on the fp32-rounded inputs,
    relative Frobenius error <= 10*k*eps32."""
    from paper_2412_01852_b200 import baseline_tol

    for i in range(2):
        A, C, S = golden[f"f{i}_A"], golden[f"f{i}_C"], golden[f"f{i}_S"]
        ref = golden[f"f{i}_rot_right_fwd_f64ref"]
        got = _gpu(A, C, S, fast=True).astype(np.float64)
        err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        assert err <= baseline_tol(C.shape[1], np.float32), err


def test_views_and_strides(cuda, oracle_mod):
    """Row-block views (ld > rows, test_variants.py:258-269) on host and device."""
    import torch

    from paper_2412_01852_b200 import apply_cuda, apply_device, generate_sequence

    big = make_matrix(300, 41, seed=2)
    guard = big.copy(order="F")
    view = big[37:250, :]
    seq = generate_sequence(41, 19, 6)
    expect = view.copy(order="F")
    oracle_mod.apply_naive(expect, seq.C, seq.S)
    apply_cuda(view, seq)
    assert_bitwise(expect, view)
    assert_bitwise(guard[:37], big[:37])
    assert_bitwise(guard[250:], big[250:])
    # device tensor with an odd leading dimension (lda = 301)
    dev = torch.empty_strided((300, 41), (1, 301), dtype=torch.float64, device=cuda)
    dev.copy_(torch.from_numpy(guard))
    apply_device(dev, seq)
    ref = guard.copy(order="F")
    oracle_mod.apply_naive(ref, seq.C, seq.S)
    assert_bitwise(ref, dev.cpu().numpy())


def test_device_tensor_and_packed_resident_mode(cuda, oracle_mod):
    import torch

    from paper_2412_01852_b200 import PackedSequence, apply_device, make_inputs

    A0, seq = make_inputs(257, 300, 37, 4)
    ref = A0.copy(order="F")
    oracle_mod.apply_naive(ref, seq.C, seq.S)
    oracle_mod.apply_naive(ref, seq.C, seq.S)
    dA = torch.from_numpy(A0.copy(order="F")).to(cuda)  # torch keeps F strides (1, m)
    assert dA.stride(0) == 1
    C = torch.from_numpy(seq.C).to(cuda)
    S = torch.from_numpy(seq.S).to(cuda)
    packed = PackedSequence((C, S), dA.shape, device=cuda)
    packed.apply(dA)
    packed.apply(dA)  # resident: the same packed coefficients, applied twice
    torch.cuda.synchronize()
    assert_bitwise(ref, dA.cpu().numpy())
    dB = torch.from_numpy(A0.copy(order="F")).to(cuda)
    apply_device(dB, (C, S))
    apply_device(dB, seq)
    assert_bitwise(ref, dB.cpu().numpy())


@pytest.mark.gpu
def test_packed_fast_only_matches_per_call_fast_path(cuda):
    """PackedSequence(fast_only=True) (rs_pack_fast_*) skips the standard records when the
    scaled form is safe: its result equals the per-call fast path bit for bit, for safe
    coefficients and for quarter turns (c = 0: standard fallback), and strict application
    of a fast-only pack is refused."""
    import torch

    from paper_2412_01852_b200 import PackedSequence, apply_device, make_inputs

    for quarter in (False, True):
        A0, seq = make_inputs(200, 150, 21, 5)
        C, S = seq.C.copy(order="F"), seq.S.copy(order="F")
        if quarter:
            C[7, 3], S[7, 3] = 0.0, 1.0
        dC, dS = torch.from_numpy(C).to(cuda), torch.from_numpy(S).to(cuda)
        dA = torch.from_numpy(A0.copy(order="F")).to(cuda)
        dB = torch.from_numpy(A0.copy(order="F")).to(cuda)
        packed = PackedSequence((dC, dS), dA.shape, device=cuda, fast_only=True)
        packed.apply(dA, fast=True)
        apply_device(dB, (dC, dS), fast=True)
        torch.cuda.synchronize()
        assert_bitwise(dB.cpu().numpy(), dA.cpu().numpy())
        with pytest.raises(ValueError, match="fast_only"):
            packed.apply(dA, fast=False)


def test_pinned_host_tensor_path(cuda, oracle_mod):
    import torch

    from paper_2412_01852_b200 import apply_cuda, make_inputs

    A0, seq = make_inputs(129, 200, 20, 9)
    ref = A0.copy(order="F")
    oracle_mod.apply_naive(ref, seq.C, seq.S)
    h = torch.empty_strided(A0.shape, (1, A0.shape[0]), dtype=torch.float64, pin_memory=True)
    h.copy_(torch.from_numpy(A0))
    apply_cuda(h, (torch.from_numpy(seq.C).pin_memory(), torch.from_numpy(seq.S).pin_memory()))
    assert_bitwise(ref, h.numpy())


def test_run_variant_and_fault_injection(cuda, oracle_mod, monkeypatch):
    """ROTSEQ_PERTURB_KERNEL=1 must make the strict comparison of the kernel path fail
    (verification.py:40-47, 76, 83); the checking algorithm (cuda-naive) is untouched."""
    from paper_2412_01852_b200 import FAULT_ENV, compare, make_inputs, run_variant

    A0, seq = make_inputs(40, 33, 8, 0)
    ref = A0.copy(order="F")
    oracle_mod.apply_naive(ref, seq.C, seq.S)
    for algo, perturbed in (("cuda", True), ("cuda-naive", False)):
        got = A0.copy(order="F")
        run_variant(algo, got, seq, threads=4, plan=None)
        assert compare(ref, got, "strict").passed
        monkeypatch.setenv(FAULT_ENV, "1")
        got = A0.copy(order="F")
        run_variant(algo, got, seq)
        assert compare(ref, got, "strict").passed is not perturbed
        monkeypatch.delenv(FAULT_ENV)


def test_zero_and_degenerate_shapes(cuda, oracle_mod):
    from paper_2412_01852_b200 import RotationSequence, apply_cuda, generate_sequence, make_inputs

    A, seq = make_inputs(0, 6, 3, 0)
    apply_cuda(A, seq)
    # identity sequence leaves A bit-identical (test_variants.py:28-33)
    A0 = make_matrix(5, 6)
    ident = RotationSequence.from_arrays(np.ones((5, 3)), np.zeros((5, 3)))
    got = A0.copy(order="F")
    apply_cuda(got, ident)
    assert_bitwise(A0, got)
    # k much larger than n - 1 (the reference's fused tier allows it, test_variants.py:121-131)
    A0 = make_matrix(5, 4)
    seq = generate_sequence(4, 9, 2)
    ref = A0.copy(order="F")
    oracle_mod.apply_naive(ref, seq.C, seq.S)
    got = A0.copy(order="F")
    apply_cuda(got, seq)
    assert_bitwise(ref, got)


def test_norm_preservation(cuda):
    """C3 (test_acceptance.py:84-101): row and Frobenius norms drift <= 100*k*eps."""
    from paper_2412_01852_b200 import make_inputs, norm_preservation_tol

    A0, seq = make_inputs(512, 700, 96, 5)
    for fast in (False, True):
        got = _gpu(A0, seq.C, seq.S, fast=fast)
        tol = norm_preservation_tol(seq.k)
        rb, ra = np.linalg.norm(A0, axis=1), np.linalg.norm(got, axis=1)
        assert np.all(np.abs(ra - rb) <= tol * rb)
        assert abs(np.linalg.norm(got) - np.linalg.norm(A0)) <= tol * np.linalg.norm(A0)


def test_explicit_q_oracle_chain(cuda, golden):
    """C2 (verification.py:198-219): vs reference_multiply(A, accumulate_q) <= 1e-12."""
    got = _gpu(golden["q_A"], golden["q_C"], golden["q_S"])
    ref = golden["q_AQ"]
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-12


def test_kernels_really_launch(cuda):
    from paper_2412_01852_b200 import _lib, make_inputs

    A0, seq = make_inputs(64, 64, 8, 0)
    n0 = _lib.launch_count()
    _gpu(A0, seq.C, seq.S)
    assert _lib.launch_count() - n0 == 2  # pack + pipeline


@pytest.mark.parametrize("chunks", ("1", "3", "8", "64"))
@pytest.mark.parametrize("side,order", SIDES_ORDERS)
def test_host_streaming_entry_point_bitwise(cuda, oracle_mod, monkeypatch, chunks, side, order):
    """rs_apply_host_* (copy-in / compute / copy-out overlapped in wave-column chunks):
    bit-identical to the oracle for any chunking, on strided host views (lda > m)."""
    from paper_2412_01852_b200 import apply_host, generate_sequence, make_inputs

    monkeypatch.setenv("RS_HOST_CHUNKS", chunks)
    m, n, k = 257, 700, 19
    A0, seq = make_inputs(m, n, k, 8)
    if side == "left":
        seq = generate_sequence(m, k, 6)
    big = np.asfortranarray(np.zeros((m + 9, n)))
    view = big[3:3 + m, :]
    view[...] = A0
    ref = A0.copy(order="F")
    oracle_mod.apply_naive(ref, seq.C, seq.S, side=side, order=order)
    apply_host(view, seq, side=side, order=order)
    assert_bitwise(ref, view, f"chunks={chunks} {side} {order}")
    assert not big[:3].any() and not big[3 + m:].any()  # rows outside the view untouched


def test_host_streaming_pinned_tensors_and_fp32(cuda, oracle_mod):
    import torch
    from paper_2412_01852_b200 import apply_host, compare, make_inputs

    m, n, k = 300, 520, 33
    A0, seq = make_inputs(m, n, k, 9)
    hA = torch.empty_strided((m, n), (1, m), dtype=torch.float64, pin_memory=True)
    hA.copy_(torch.from_numpy(A0))
    hC = torch.from_numpy(np.asfortranarray(seq.C)).pin_memory()
    hS = torch.from_numpy(np.asfortranarray(seq.S)).pin_memory()
    ref = A0.copy(order="F")
    oracle_mod.apply_naive(ref, seq.C, seq.S)
    apply_host(hA, (hC, hS), fast=True)
    assert compare(ref, hA.numpy(), "baseline", k=k).passed
    A32 = np.asfortranarray(A0.astype(np.float32))
    apply_host(A32, (seq.C.astype(np.float32), seq.S.astype(np.float32)), fast=True)
    ref32 = oracle_mod.upcast_reference(A0.astype(np.float32), seq.C.astype(np.float32), seq.S.astype(np.float32))
    assert np.linalg.norm(A32 - ref32) / np.linalg.norm(ref32) <= 10 * k * np.finfo(np.float32).eps


def test_cli_run_and_verify(cuda, tmp_path):
    """``python -m paper_2412_01852_b200.cli``: run writes the reference's CSV (and the
    extended columns with the kernel's peak fraction) and verifies small cases against
    cuda-naive; verify runs the criterion-1 grid bit for bit."""
    from paper_2412_01852_b200 import cli

    out = tmp_path / "run.csv"
    assert cli.main(["run", "--algo", "cuda", "--n", "96", "--m", "70", "--k", "9", "--reps", "2",
                     "--csv", str(out), "--csv-extended", "--strict-arith", "on"]) == 0
    lines = out.read_text().splitlines()
    assert lines[0] == "n,Flops,algo,m,k,threads,reps,seconds,verified,kernel_seconds,peak_frac"
    assert lines[1].split(",")[8] == "True"
    out2 = tmp_path / "sweep.csv"
    assert cli.main(["run", "--sweep", "64", "128", "--k", "12", "--reps", "1", "--csv", str(out2)]) == 0
    assert out2.read_text().splitlines()[0] == "n,Flops" and len(out2.read_text().splitlines()) == 3
    assert cli.main(["verify", "--quick"]) == 0


@pytest.mark.parametrize("kind", ("rotation", "reflector"))
def test_fp32_wide_window(cuda, oracle_mod, monkeypatch, kind):
    """fp32 right-side launches with units of >= 9 sweeps run the 16-sweep window
    (rs_plan_info band_width 16): strict is bit-identical to the numpy fp32 oracle and to
    the 8-sweep window (RS_F32_K8=1), in forced multi-round / multi-CTA geometries too;
    fast stays within 10*k*eps32 of the fp64 reference on the fp32 inputs."""
    from paper_2412_01852_b200 import _lib

    if _lib.plan_info(130, 300, 16, dtype=_lib.DTYPE_F32)["band_width"] != 16:
        pytest.skip("library built without the 16-sweep window (RS_F32_WIDE=0, the default)")
    for (m, n, k, order) in ((130, 300, 16, "forward"), (64, 100, 18, "reverse"), (300, 77, 40, "forward"),
                             (97, 260, 129, "reverse"), (200, 60, 32, "forward")):
        assert _lib.plan_info(m, n, k, dtype=_lib.DTYPE_F32)["band_width"] == 16, (m, n, k)
        rng = np.random.Generator(np.random.Philox(k))
        A = np.asfortranarray(rng.uniform(-1, 1, (m, n)).astype(np.float32))
        th = rng.uniform(0, 2 * np.pi, (n - 1, k))
        C, S = np.cos(th).astype(np.float32), np.sin(th).astype(np.float32)
        ref = A.copy(order="F")
        oracle_mod.numpy_apply_naive(ref, C, S, order=order, kind=kind)
        for mw, grid in (("", ""), ("4", "3"), ("1", "")):
            for key, val in (("RS_DEBUG_MAX_WARPS", mw), ("RS_DEBUG_GRID", grid)):
                if val:
                    monkeypatch.setenv(key, val)
                else:
                    monkeypatch.delenv(key, raising=False)
            assert_bitwise(ref, _gpu(A, C, S, order=order, kind=kind), f"wide fp32 {m}x{n} k={k} mw={mw} grid={grid}")
        monkeypatch.delenv("RS_DEBUG_MAX_WARPS", raising=False)
        monkeypatch.delenv("RS_DEBUG_GRID", raising=False)
        monkeypatch.setenv("RS_F32_K8", "1")
        assert _lib.plan_info(m, n, k, dtype=_lib.DTYPE_F32)["band_width"] == 8
        assert_bitwise(ref, _gpu(A, C, S, order=order, kind=kind), "8-sweep window")
        monkeypatch.delenv("RS_F32_K8")
        ref64 = oracle_mod.upcast_reference(A, C, S, order=order, kind=kind)
        got = _gpu(A, C, S, order=order, kind=kind, fast=True).astype(np.float64)
        err = np.linalg.norm(got - ref64) / np.linalg.norm(ref64)
        assert err <= 10 * k * np.finfo(np.float32).eps, (m, n, k, err)

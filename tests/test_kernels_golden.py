"""Micro-kernel API (kernel_wave_apply / kernel_edge_apply, kernels.py:335-410).

CPU: the oracle's restatement reproduces the reference's own outputs bit for bit
(tests/golden/golden_kernels_v1.npz, written by tests/golden/make_golden_kernels.py),
and the host-side argument checks raise the reference's errors before any GPU work.
GPU (-m gpu): the CUDA micro-kernel (rs_wave_apply_*) through the mirror API matches
the same goldens bitwise in strict mode and within 10*k_r*n_waves*eps in fast mode;
edge + pipeline passes equal the plain loop (test_kernels.py:181-203).
"""

from __future__ import annotations

import os
import warnings

import numpy as np
import pytest

from conftest import HERE, assert_bitwise

GOLDEN_K = os.path.join(HERE, "golden", "golden_kernels_v1.npz")


@pytest.fixture(scope="module")
def gk():
    return np.load(GOLDEN_K)


def _wave_cases(gk):
    i = 0
    while f"wave{i}_meta" in gk:
        yield i, [int(x) for x in gk[f"wave{i}_meta"]]
        i += 1


def _edge_cases(gk):
    i = 0
    while f"edge{i}_meta" in gk:
        yield i, [int(x) for x in gk[f"edge{i}_meta"]]
        i += 1


@pytest.mark.parametrize("kind", ["rotation", "reflector"])
def test_oracle_wave_apply_matches_reference(gk, kind):
    from oracle import oracle

    for i, (m_r, k_r, n_cols, n_waves, col0) in _wave_cases(gk):
        P = gk[f"wave{i}_panel"].copy()
        oracle.wave_apply(P, gk[f"wave{i}_ct"], gk[f"wave{i}_st"], n_waves, k_r, col0, kind)
        assert_bitwise(gk[f"wave{i}_{kind}"], P, f"wave case {i}")


@pytest.mark.parametrize("kind", ["rotation", "reflector"])
@pytest.mark.parametrize("tri", ["startup", "shutdown"])
def test_oracle_edge_apply_matches_reference(gk, kind, tri):
    from oracle import oracle
    from paper_2412_01852_b200.kernels import edge_traversal

    for i, (m_r, n, k_chunk, p0, k) in _edge_cases(gk):
        P = gk[f"edge{i}_panel"].copy()
        oracle.edge_apply(P, gk[f"edge{i}_C"], gk[f"edge{i}_S"], p0, k_chunk, tri, kind)
        assert_bitwise(gk[f"edge{i}_{tri}_{kind}"], P, f"edge case {i}")
        order = np.array(list(edge_traversal(n, k_chunk, tri)), dtype=np.int64).reshape(-1, 2)
        assert np.array_equal(order, gk[f"edge{i}_{tri}_order"])


def test_kernel_api_argument_checks():
    """Reference messages (kernels.py:325-360), raised before any GPU call."""
    from paper_2412_01852_b200.kernels import KernelShape, PanelView, kernel_edge_apply, kernel_wave_apply

    with pytest.raises(ValueError, match="positive"):
        KernelShape(0, 2)
    with pytest.raises(ValueError, match="mode"):
        KernelShape(4, 2, mode="turbo")
    shape = KernelShape(4, 2)
    ct = np.ones(20)
    with pytest.raises(ValueError, match="C-contiguous"):
        kernel_wave_apply(np.zeros((10, 4), order="F"), ct, ct, 3, shape)
    with pytest.raises(ValueError, match="rows"):
        kernel_wave_apply(np.zeros((10, 5)), ct, ct, 3, shape)
    with pytest.raises(ValueError, match="usable columns"):
        kernel_wave_apply(np.zeros((4, 4)), ct, ct, 3, shape)
    with pytest.raises(ValueError, match="shorter"):
        kernel_wave_apply(np.zeros((10, 4)), ct[:3], ct[:3], 3, shape)
    with pytest.raises(ValueError, match="triangle"):
        kernel_edge_apply(np.zeros((10, 4)), np.ones((9, 2)), np.ones((9, 2)), 0, 2, "middle", shape)
    buf = np.arange(40.0)
    v = PanelView(base=8, n_cols=4, m_r=4)
    assert np.array_equal(v.as_array(buf), buf[8:24].reshape(4, 4))


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["rotation", "reflector"])
def test_gpu_wave_apply_matches_reference(cuda, gk, kind):
    from paper_2412_01852_b200 import compare
    from paper_2412_01852_b200.kernels import KernelShape, kernel_wave_apply

    for i, (m_r, k_r, n_cols, n_waves, col0) in _wave_cases(gk):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            shape = KernelShape(m_r, k_r)
        P = gk[f"wave{i}_panel"].copy()
        kernel_wave_apply(P, gk[f"wave{i}_ct"], gk[f"wave{i}_st"], n_waves, shape, kind, col0)
        assert_bitwise(gk[f"wave{i}_{kind}"], P, f"wave case {i} strict")
        P = gk[f"wave{i}_panel"].copy()
        kernel_wave_apply(P, gk[f"wave{i}_ct"], gk[f"wave{i}_st"], n_waves, KernelShape(m_r, k_r, mode="fast"),
                          kind, col0)
        rep = compare(gk[f"wave{i}_{kind}"], P, "baseline", k=n_waves * k_r)
        assert rep.passed, f"wave case {i} fast: {rep}"


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["rotation", "reflector"])
def test_gpu_edge_apply_matches_reference(cuda, gk, kind):
    import torch

    from paper_2412_01852_b200.kernels import KernelShape, kernel_edge_apply

    for i, (m_r, n, k_chunk, p0, k) in _edge_cases(gk):
        for tri in ("startup", "shutdown"):
            P = gk[f"edge{i}_panel"].copy()
            kernel_edge_apply(P, gk[f"edge{i}_C"], gk[f"edge{i}_S"], p0, k_chunk, tri, KernelShape(m_r, 1), kind)
            assert_bitwise(gk[f"edge{i}_{tri}_{kind}"], P, f"edge case {i} {tri}")
            # device-resident panel (torch, in place)
            dP = torch.from_numpy(gk[f"edge{i}_panel"].copy()).cuda()
            kernel_edge_apply(dP, gk[f"edge{i}_C"], gk[f"edge{i}_S"], p0, k_chunk, tri, KernelShape(m_r, 1), kind)
            assert_bitwise(gk[f"edge{i}_{tri}_{kind}"], dP.cpu().numpy(), f"edge case {i} {tri} (device)")


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["rotation", "reflector"])
def test_gpu_edge_plus_waves_equal_naive(cuda, oracle_mod, kind):
    """One k-chunk as startup triangle + full-width waves + shutdown triangle equals the
    plain loop on the panel (the reference's test_kernels.py:181-203 composition)."""
    from paper_2412_01852_b200 import make_inputs
    from paper_2412_01852_b200.kernels import KernelShape, kernel_edge_apply, kernel_wave_apply

    m_r, n, k = 16, 24, 4
    A0, seq = make_inputs(m_r, n, k, 9)
    ref = A0.copy(order="F")
    oracle_mod.apply_naive(ref, seq.C, seq.S, kind=kind)
    panel = np.ascontiguousarray(A0.T)  # (n_cols, m_r), column j contiguous
    kernel_edge_apply(panel, seq.C, seq.S, 0, k, "startup", KernelShape(m_r, 1), kind)
    n_waves = n - k  # waves t0 = k-1 .. n-2, each with all k lanes
    ct = np.empty(n_waves * k)
    st = np.empty(n_waves * k)
    for w in range(n_waves):
        for lane in range(k):
            j = w + k - 1 - lane  # the pair lane `lane` rotates in wave w (col0 = 0)
            ct[w * k + lane] = seq.C[j, lane]
            st[w * k + lane] = seq.S[j, lane]
    kernel_wave_apply(panel, ct, st, n_waves, KernelShape(m_r, k), kind, 0)
    kernel_edge_apply(panel, seq.C, seq.S, 0, k, "shutdown", KernelShape(m_r, 1), kind)
    assert_bitwise(ref, np.asfortranarray(panel.T), "edge + waves vs naive")

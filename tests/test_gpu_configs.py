"""BASELINE.json configs 1-5 at full size on the GPU.

Full-size parity uses what the domain allows: rows (right side) / columns (left
side) are independent, so a seeded subset of owners is checked bit for bit against
the CPU oracle in strict mode, and the whole matrix is checked through
size-independent properties (norm preservation, GPU-count/shard invariance, strict
vs. fast within 10*k*eps). Config 2 is compared in full against the oracle's
kernel tier on all host cores."""

from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import assert_bitwise

pytestmark = pytest.mark.gpu


def _threads():
    return len(os.sched_getaffinity(0))


def _device_apply(A, C, S, w, fast):
    import torch

    from paper_2412_01852_b200 import apply_device

    tdt = torch.float64 if A.dtype == np.float64 else torch.float32
    dA = torch.empty_strided(A.shape, (1, A.shape[0]), dtype=tdt, device="cuda")
    dA.copy_(torch.from_numpy(A))
    apply_device(dA, (torch.from_numpy(C).to(tdt), torch.from_numpy(S).to(tdt)), fast=fast, side=w.side,
                 order=w.order)
    return dA.cpu().numpy()


def _owner_subset(n_owners, count, seed=0):
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(n_owners, size=min(count, n_owners), replace=False))
    return idx


def _oracle_subset(oracle_mod, w, A, C, S, idx):
    """Oracle on the selected owners only (rows independent on the right side,
    columns on the left)."""
    sub = np.asfortranarray(A[:, idx] if w.side.value == "left" else A[idx, :]).astype(np.float64)
    oracle_mod.apply_naive(sub, C.astype(np.float64), S.astype(np.float64), side=w.side.value,
                           order=w.order.value)
    return sub


def _take(X, w, idx):
    return np.asfortranarray(X[:, idx] if w.side.value == "left" else X[idx, :])


def test_config1_exact(cuda, oracle_mod):
    from paper_2412_01852_b200 import WORKLOADS, compare, make_workload_inputs

    w = WORKLOADS[1]
    A, C, S = make_workload_inputs(w)
    ref = A.copy(order="F")
    oracle_mod.apply_naive(ref, C, S)
    assert_bitwise(ref, _device_apply(A, C, S, w, fast=False))
    assert compare(ref, _device_apply(A, C, S, w, fast=True), "baseline", k=w.k).passed


def test_config2_full_matrix(cuda, oracle_mod):
    from paper_2412_01852_b200 import WORKLOADS, compare, make_workload_inputs

    w = WORKLOADS[2]
    A, C, S = make_workload_inputs(w)
    ref = A.copy(order="F")
    oracle_mod.apply_blocked(ref, C, S, threads=_threads())  # strict kernel tier == naive bitwise
    assert_bitwise(ref, _device_apply(A, C, S, w, fast=False), "config 2 strict")
    rep = compare(ref, _device_apply(A, C, S, w, fast=True), "baseline", k=w.k)
    assert rep.passed, rep


@pytest.mark.parametrize("cfg", (3, 4, 5))
def test_full_size_subset_parity_and_invariants(cuda, oracle_mod, cfg):
    import torch

    from paper_2412_01852_b200 import WORKLOADS, baseline_tol, make_workload_inputs, shard_range

    w = WORKLOADS[cfg]
    A, C, S = make_workload_inputs(w)
    strict = _device_apply(A, C, S, w, fast=False)
    fast = _device_apply(A, C, S, w, fast=True)
    idx = _owner_subset(w.owners, 96 if cfg != 5 else 48, seed=cfg)
    # 1. strict, subset of owners, bit for bit (fp32: the numpy fp32 oracle)
    if w.dtype == np.float64:
        ref = _oracle_subset(oracle_mod, w, A, C, S, idx)
        assert_bitwise(ref, _take(strict, w, idx), f"config {cfg} strict subset")
    else:
        sub = _take(A, w, idx)
        oracle_mod.numpy_apply_naive(sub, C, S, side=w.side.value, order=w.order.value)
        assert_bitwise(sub, _take(strict, w, idx), "config 4 strict fp32 subset")
        ref = _oracle_subset(oracle_mod, w, A, C, S, idx)  # fp64 reference on fp32 inputs
    # 2. fast, subset, within BASELINE's 10*k*eps of the working dtype
    got = _take(fast, w, idx).astype(np.float64)
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert err <= baseline_tol(w.k, w.dtype), err
    # 3. whole matrix: strict vs fast within tolerance; norm preservation (100*k*eps)
    X, Y = strict.astype(np.float64), fast.astype(np.float64)
    assert np.linalg.norm(X - Y) / np.linalg.norm(X) <= baseline_tol(w.k, w.dtype)
    eps = float(np.finfo(w.dtype).eps)
    nA = np.linalg.norm(A.astype(np.float64))
    assert abs(np.linalg.norm(X) - nA) <= 100 * w.k * eps * nA
    # 4. GPU-count invariance: 8 shards applied separately == the whole, bitwise
    parts = []
    for r in range(8):
        o0, o1 = shard_range(w.owners, 8, r)
        sh = np.asfortranarray(A[:, o0:o1] if w.side.value == "left" else A[o0:o1, :])
        parts.append(_device_apply(sh, C, S, w, fast=False))
    whole = np.concatenate(parts, axis=1 if w.side.value == "left" else 0)
    assert_bitwise(strict, np.asfortranarray(whole), f"config {cfg} shard invariance")
    torch.cuda.empty_cache()


@pytest.mark.parametrize("m,n,k,side,dtype", [
    (512, 512, 64, 0, 0), (4096, 4096, 192, 0, 0), (65536, 2048, 256, 0, 0), (8192, 8192, 128, 0, 1),
    (16384, 16384, 96, 1, 0), (8192, 2048, 256, 0, 0), (16384, 2048, 256, 0, 0), (32768, 2048, 256, 0, 0),
    (4096, 4096, 192, 1, 0), (4096, 4096, 192, 0, 1),  # left side keeps the aligned plan; fp32 takes equal chains
])
def test_launch_plan_matches_schedule_model(cuda, m, n, k, side, dtype):
    """plan_launch (C++) and the schedule model whose hand-off protocol the CPU suite
    simulates for deadlock freedom (tests/pipeline_model.py) pick the same launch: grid,
    warps per CTA and unit count, including the aligned plans."""
    import torch

    from paper_2412_01852_b200 import _lib
    from pipeline_model import Geometry, plan, warp_cap

    if torch.cuda.get_device_properties(0).multi_processor_count != 148:
        pytest.skip("model parameters are for a 148-SM B200")
    left = side == 1
    tsz = 8 if dtype == 0 else 4
    cap = warp_cap(tsz, S=2, max_warps=12 if left else 16, left=left)
    owners, length = (n, m) if left else (m, n)
    pl = plan(Geometry(owners=owners, length=length, k=k), cap=cap, left=left)
    info = _lib.plan_info(m, n, k, side=side, dtype=dtype)
    assert (info["grid_ctas"], info["warps_per_cta"], info["units"]) == (pl["G"], pl["NW"], pl["U"])


@pytest.mark.parametrize("m,n,k,side", [
    (16384, 2048, 256, "right"),  # aligned plan, 4 rounds per CTA
    (8192, 2048, 256, "right"),   # aligned plan, 2 rounds
    (2048, 8192, 96, "left"),     # left side, aligned plan (one chain per CTA round)
])
def test_aligned_plans_bitwise_vs_naive_kernel(cuda, m, n, k, side):
    """Aligned launch plans (uniform unit widths, chains filling CTA rounds) in strict
    arithmetic equal the independent one-thread-per-owner GPU kernel bit for bit."""
    import torch

    from paper_2412_01852_b200 import apply_device

    g = torch.Generator(device="cpu").manual_seed(11)
    A = torch.randn(n, m, dtype=torch.float64, generator=g).to(cuda).t()  # column-major m x n
    ln = m if side == "left" else n
    th = torch.rand(k, ln - 1, dtype=torch.float64, generator=g).t() * 6.283185307179586
    C, S = torch.cos(th).to(cuda), torch.sin(th).to(cuda)
    B = A.clone(memory_format=torch.preserve_format)
    apply_device(A, (C, S), fast=False, side=side)
    apply_device(B, (C, S), fast=False, side=side, algo="naive")
    torch.cuda.synchronize()
    assert_bitwise(B.cpu().numpy(), A.cpu().numpy())


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ("rotation", "reflector"))
def test_equal_chain_plan_bitwise_and_fast_tolerance(cuda, kind):
    """The equal-chain plan (chains of 27 units of 7-8 sweeps on 144 CTAs, sweep-split
    offset; what config 2's shape selects on a 148-SM B200) against the independent
    one-thread-per-owner kernel: strict bitwise, fast within 10 k eps; and with the plan
    switched off (RS_NO_EQUAL_CHAIN=1: the aligned plan) bit-identical strict results."""
    import os

    import torch

    from paper_2412_01852_b200 import _lib, apply_device

    if torch.cuda.get_device_properties(0).multi_processor_count != 148:
        pytest.skip("the plan under test is chosen for a 148-SM B200")
    m, n, k = 4096, 2304, 192   # 64 tiles x 192 sweeps: the same unit split as config 2
    info = _lib.plan_info(m, n, k)
    assert (info["grid_ctas"], info["warps_per_cta"], info["units"]) == (144, 12, 1728)
    g = torch.Generator(device="cpu").manual_seed(5)
    A0 = torch.randn(n, m, dtype=torch.float64, generator=g).to(cuda).t()
    th = torch.rand(k, n - 1, dtype=torch.float64, generator=g).t() * 6.283185307179586
    C, S = torch.cos(th).to(cuda), torch.sin(th).to(cuda)
    ref = A0.clone(memory_format=torch.preserve_format)
    apply_device(ref, (C, S), fast=False, kind=kind, algo="naive")
    got = A0.clone(memory_format=torch.preserve_format)
    apply_device(got, (C, S), fast=False, kind=kind)
    torch.cuda.synchronize()
    assert_bitwise(ref.cpu().numpy(), got.cpu().numpy())
    fast = A0.clone(memory_format=torch.preserve_format)
    apply_device(fast, (C, S), fast=True, kind=kind)
    torch.cuda.synchronize()
    rel = (torch.linalg.norm(fast - ref) / torch.linalg.norm(ref)).item()
    assert rel <= 10 * k * 2.220446049250313e-16, rel
    os.environ["RS_NO_EQUAL_CHAIN"] = "1"
    try:
        assert _lib.plan_info(m, n, k)["grid_ctas"] == 128
        alt = A0.clone(memory_format=torch.preserve_format)
        apply_device(alt, (C, S), fast=False, kind=kind)
        torch.cuda.synchronize()
    finally:
        del os.environ["RS_NO_EQUAL_CHAIN"]
    assert_bitwise(ref.cpu().numpy(), alt.cpu().numpy())

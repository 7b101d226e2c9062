"""Shared fixtures. GPU tests are marked ``@pytest.mark.gpu``; everything else runs on
CPU. Helpers mirror the reference suite's conftest (pkg/tests/conftest.py:7-50)."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)

GOLDEN = os.path.join(HERE, "golden", "golden_v1.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running (full-size BASELINE configs)")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle

    oracle.build()
    return oracle


def make_matrix(m: int, n: int, seed: int = 0) -> np.ndarray:
    """conftest.py:7-9 of the reference."""
    rng = np.random.Generator(np.random.Philox(seed))
    return np.asfortranarray(rng.standard_normal((m, n)))


def assert_bitwise(expected: np.ndarray, got: np.ndarray, msg: str = ""):
    """conftest.py:16-23 of the reference (uint view comparison)."""
    expected = np.ascontiguousarray(expected)
    got = np.ascontiguousarray(got)
    view = np.uint64 if expected.dtype == np.float64 else np.uint32
    if expected.shape != got.shape or not np.array_equal(expected.view(view), got.view(view)):
        diff = np.abs(expected.astype(np.float64) - got.astype(np.float64))
        idx = np.unravel_index(np.argmax(diff), diff.shape) if diff.size else ()
        pytest.fail(f"not bit-identical {msg}: max |diff| {diff.max() if diff.size else 0:.3e} at {idx}")


def assert_naive_equivalent_order(order, n: int, k: int):
    """conftest.py:26-43 of the reference: an order is exchangeable with the plain
    loop iff, per column, transforms touching it appear in plain-order positions, and
    the multiset matches exactly."""
    last = {}
    count = 0
    for q, p in order:
        assert 0 <= q <= n - 2 and 0 <= p <= k - 1, f"(q={q}, p={p}) out of range"
        key = p * (n - 1) + q
        for col in (q, q + 1):
            prev = last.get(col, -1)
            assert prev < key, f"column {col}: transform (q={q}, p={p}) after a later plain-order transform"
            last[col] = key
        count += 1
    assert count == (n - 1) * k, f"applied {count} transforms, want {(n - 1) * k}"


def gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # noqa: BLE001
        return False


@pytest.fixture(scope="session")
def cuda():
    if not gpu_available():
        pytest.fail("GPU test run without a CUDA device (run -m \"not gpu\" on CPU)")
    import torch

    torch.cuda.set_device(0)
    from paper_2412_01852_b200 import _lib

    _lib.load()  # fails loudly if the extension is missing
    return torch.device("cuda", 0)

"""The tile model (paper_2412_01852_b200/model.py, the counterpart of the reference's
memops_kernel / choose_block_sizes, rotseq/model.py:97-108 and blocking.py:115-147) and
its pin to the library's compile-time tile shape (rs_tile_shape, no GPU needed)."""

import pytest

from paper_2412_01852_b200 import _lib, model as M


def test_memops_window_matches_the_reference_formula_shape():
    # reference kernel tier: (2/k_r + 2/n_b + 2/m_r) per applied transform (model.py:97-108)
    r = M.memops_window(K=8, R=2, k=192)
    assert r.shared == pytest.approx(2 / 8)            # 2/k_r: one column in, one out per wave
    assert r.coefficient == pytest.approx(2 / 64)      # 2/m_r with m_r = 32 R rows per warp
    assert r.hbm == pytest.approx(2 / 192)             # A crosses HBM once per ring-linked chain
    assert r.per_rotation_factor == pytest.approx(2 / 8 + 2 / 64 + 2 / 192)
    # chains cut into 12-unit pieces (one CTA round) cross HBM once per 96 sweeps
    assert M.memops_window(8, 2, 192, ring_linked_units=12).hbm == pytest.approx(2 / 96)
    # monotone: a wider window and more rows per thread both lower the traffic
    assert M.memops_window(16, 2, 192).per_rotation_factor < r.per_rotation_factor
    assert M.memops_window(8, 4, 192).per_rotation_factor < r.per_rotation_factor
    with pytest.raises(ValueError):
        M.memops_window(0, 2, 8)


def test_issue_cycles_terms():
    c = M.issue_cycles(8, 2, 8, "scaled")
    # 2 DFMA per transform element; 28% of them find their multiplier in the reuse cache
    assert c["fp"] == pytest.approx(2 * (0.28 * 2 + 0.72 * 3))
    assert c["smem"] == pytest.approx((2 + 2) / 8)
    assert c["coef"] == pytest.approx(0.5)
    assert c["total"] == pytest.approx(c["fp"] + c["smem"] + c["coef"] + c["protocol"])
    # the forms order as measured: scaled < fast standard < strict
    assert c["total"] < M.issue_cycles(8, 2, 8, "fast")["total"] < M.issue_cycles(8, 2, 8, "strict")["total"]
    # more rows per thread amortise the coefficient load and the register-file reads
    assert M.issue_cycles(8, 3, 8)["total"] < c["total"]


def test_budgets_reject_the_shapes_that_were_measured_to_lose():
    tab = {(c["K"], c["R"], c["warps"]): c for c in M.candidate_table(8)}
    assert tab[(8, 2, 12)]["feasible"]
    # R = 3 does not fit 168 registers (measured: spills, no gain); 8-warp CTAs have the
    # registers but two warps per SMSP cannot cover the hand-off waits (measured: -30%)
    assert "registers" in tab[(8, 3, 12)]["why"]
    assert "warps per SMSP" in tab[(8, 4, 8)]["why"]
    # the 16-sweep window: its unrolled block outgrows the instruction cache (ncu: 62%
    # no_instruction stalls for the fp32 build) and the shared memory
    assert "block body" in tab[(16, 2, 12)]["why"]
    tab32 = {(c["K"], c["R"], c["warps"]): c for c in M.candidate_table(4)}
    assert "block body" in tab32[(16, 2, 12)]["why"]


@pytest.mark.parametrize("dtype,tsz", [(_lib.DTYPE_F64, 8), (_lib.DTYPE_F32, 4)])
@pytest.mark.parametrize("side,left", [(_lib.SIDE_RIGHT, False), (_lib.SIDE_LEFT, True)])
def test_library_tile_shape_is_the_models_choice(dtype, tsz, side, left):
    built = _lib.tile_shape(dtype, side)
    want = M.choose_tile_shape(tsz, left)
    assert built["window_sweeps"] == want.K
    assert built["rows_per_thread"] == want.R
    assert built["ring_chunks"] == want.ring_chunks
    # the register budget the shape was chosen for: the dedicated <= 12-warp build where
    # the family has one, else the family's only build
    budget_warps = built["small_cta_warps"] or built["max_warps"]
    assert budget_warps == want.warps
    # the largest CTA follows from shared memory alone (multiples of 4 warps, at most 16)
    per = M.smem_per_warp(want.K, want.R, tsz, want.ring_chunks, left)
    cap = min(16, (M.SmSpec().smem_optin_bytes - (want.ring_chunks + 3) * 8) // per) & ~3
    assert built["max_warps"] <= cap


def test_modelled_throughput_brackets_the_measured_body():
    # body_r.cu (block body alone, no protocol): 33.2 counted TF/s at K=8, R=2, 12 warps
    s = M.TileShape(8, 2, 12)
    assert 30.0 < M.modelled_tflops(s, 8) < 36.0

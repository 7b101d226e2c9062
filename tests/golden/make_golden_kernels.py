"""Golden vectors for the micro-kernel API, produced by the REFERENCE itself.

Run in the build container (where the read-only reference lives):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden_kernels.py

Writes tests/golden/golden_kernels_v1.npz. Only the reference's public API is called:
``kernels.kernel_wave_apply`` (kernels.py:335-371; generic and fixed-shape kernels,
strict build), ``kernels.kernel_edge_apply`` (kernels.py:374-410) and
``kernels.edge_traversal`` (kernels.py:413-422). Inputs are Philox-seeded.
"""

from __future__ import annotations

import os
import sys
import warnings

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_kernels_v1.npz")

# (m_r, k_r, n_cols, n_waves, col0): the four fixed shapes, generic shapes, col0 offsets
WAVE_CASES = [
    (16, 2, 40, 30, 0), (12, 3, 33, 25, 2), (8, 5, 50, 40, 1), (48, 1, 20, 19, 0),
    (7, 4, 30, 20, 3), (1, 1, 2, 1, 0), (33, 6, 64, 50, 5), (5, 8, 41, 33, 0),
]
# (m_r, n, k_chunk, p0, k): kernel_edge_apply startup + shutdown triangles
EDGE_CASES = [(16, 12, 4, 0, 4), (8, 9, 3, 2, 6), (5, 30, 8, 1, 10)]


def main():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, REF)
    from rotseq.core import TransformKind  # noqa: PLC0415
    from rotseq.kernels import KernelShape, edge_traversal, kernel_edge_apply, kernel_wave_apply  # noqa: PLC0415

    out = {}
    for ci, (m_r, k_r, n_cols, n_waves, col0) in enumerate(WAVE_CASES):
        rng = np.random.Generator(np.random.Philox(100 + ci))
        panel = np.ascontiguousarray(rng.standard_normal((n_cols, m_r)))
        th = rng.uniform(0.0, 2.0 * np.pi, size=n_waves * k_r)
        ct, st = np.cos(th), np.sin(th)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            shape = KernelShape(m_r, k_r)
        out[f"wave{ci}_panel"] = panel.copy()
        out[f"wave{ci}_ct"] = ct
        out[f"wave{ci}_st"] = st
        out[f"wave{ci}_meta"] = np.array([m_r, k_r, n_cols, n_waves, col0])
        for kind in (TransformKind.ROTATION, TransformKind.REFLECTOR):
            got = panel.copy()
            kernel_wave_apply(got, ct, st, n_waves, shape, kind, col0)
            out[f"wave{ci}_{kind.value}"] = got
            gen = panel.copy()
            kernel_wave_apply(gen, ct, st, n_waves, shape, kind, col0, force_generic=True)
            assert np.array_equal(gen.view(np.uint64), got.view(np.uint64))
    for ci, (m_r, n, k_chunk, p0, k) in enumerate(EDGE_CASES):
        rng = np.random.Generator(np.random.Philox(200 + ci))
        panel = np.ascontiguousarray(rng.standard_normal((n, m_r)))
        th = rng.uniform(0.0, 2.0 * np.pi, size=(n - 1, k))
        C, S = np.asfortranarray(np.cos(th)), np.asfortranarray(np.sin(th))
        shape = KernelShape(m_r, 1)
        out[f"edge{ci}_panel"] = panel.copy()
        out[f"edge{ci}_C"] = C
        out[f"edge{ci}_S"] = S
        out[f"edge{ci}_meta"] = np.array([m_r, n, k_chunk, p0, k])
        for tri in ("startup", "shutdown"):
            for kind in (TransformKind.ROTATION, TransformKind.REFLECTOR):
                got = panel.copy()
                kernel_edge_apply(got, C, S, p0, k_chunk, tri, shape, kind)
                out[f"edge{ci}_{tri}_{kind.value}"] = got
            out[f"edge{ci}_{tri}_order"] = np.array(list(edge_traversal(n, k_chunk, tri)), dtype=np.int64).reshape(-1, 2)
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT}: {len(out)} arrays")


if __name__ == "__main__":
    main()

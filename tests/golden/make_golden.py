"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (where the read-only reference lives):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Writes tests/golden/golden_v1.npz. The reference (package ``rotseq``) is imported
from /root/reference/pkg/src and only its public API is called:
``verification.make_inputs`` (verification.py:102-105), ``core.generate_sequence``
(core.py:94-107), ``core.apply_naive`` strict (core.py:365-374),
``blocking.apply_blocked`` (blocking.py:420-476), ``oracle.accumulate_q`` /
``oracle.reference_multiply`` (oracle.py:102-136).

Extensions the reference does not define are generated with the reference
through exact identities:
  left side      : apply_naive on A^T (F-order copy), transposed back;
  reverse order  : apply_naive on the column-mirrored A with mirrored C/S and
                   S negated (rotation) or C negated (reflector), un-mirrored;
  fp32           : apply_naive in fp64 on the fp32-rounded A, C, S
                   (from_arrays(..., check_orthonormal=False)).
Nothing here reads or writes outside the repo except importing the reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_v1.npz")


def main():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, REF)
    from rotseq.blocking import apply_blocked  # noqa: PLC0415
    from rotseq.core import RotationSequence, TransformKind, apply_naive, generate_sequence  # noqa: PLC0415
    from rotseq.oracle import accumulate_q, reference_multiply  # noqa: PLC0415
    from rotseq.verification import default_plan, default_shape, make_inputs  # noqa: PLC0415

    R, H = TransformKind.ROTATION, TransformKind.REFLECTOR
    data = {}

    def naive(A, seq, kind):
        out = np.asfortranarray(A.copy())
        apply_naive(out, seq, kind)
        return out

    def right(A, C, S, kind, check=True):
        return naive(A, RotationSequence.from_arrays(C, S, check_orthonormal=check), kind)

    def left(A, C, S, kind, check=True):
        return np.asfortranarray(right(np.asfortranarray(A.T), C, S, kind, check).T)

    def reverse(A, C, S, kind, side_fn, axis, check=True):
        Am = np.flip(A, axis=axis)
        Cm, Sm = C[::-1, :], S[::-1, :]
        if kind is R:
            Cm, Sm = Cm, -Sm
        else:
            Cm, Sm = -Cm, Sm
        out = side_fn(np.asfortranarray(Am), Cm, Sm, kind, check)
        return np.asfortranarray(np.flip(out, axis=axis))

    cases = [(1, 2, 1, 0), (2, 4, 1, 7), (3, 9, 3, 7), (5, 6, 3, 0), (17, 33, 8, 7), (33, 40, 9, 0),
             (64, 64, 12, 7), (129, 64, 5, 7), (257, 33, 12, 7), (40, 48, 6, 0), (16, 400, 180, 9),
             (70, 17, 30, 3), (31, 3, 7, 5)]
    data["cases"] = np.array(cases, dtype=np.int64)
    for idx, (m, n, k, seed) in enumerate(cases):
        A0, seq = make_inputs(m, n, k, seed)
        key = f"c{idx}"
        data[f"{key}_A"] = A0
        data[f"{key}_C"] = seq.C
        data[f"{key}_S"] = seq.S
        for kname, kind in (("rot", R), ("refl", H)):
            data[f"{key}_{kname}_right_fwd"] = naive(A0, seq, kind)
            data[f"{key}_{kname}_right_rev"] = reverse(A0, seq.C, seq.S, kind, right, axis=1)
            # left side needs (m-1) x k coefficients: a sequence of its own from seed+2
            if m >= 2:
                sl = generate_sequence(m, k, seed + 2)
                data[f"{key}_Cl"] = sl.C
                data[f"{key}_Sl"] = sl.S
                data[f"{key}_{kname}_left_fwd"] = left(A0, sl.C, sl.S, kind)
                data[f"{key}_{kname}_left_rev"] = reverse(A0, sl.C, sl.S, kind, left, axis=0)
        # the reference's kernel tier (strict) on the same case: must equal naive bitwise
        if m >= 1:
            got = np.asfortranarray(A0.copy())
            shape = default_shape()
            apply_blocked(got, seq, default_plan(shape), shape, threads=2)
            data[f"{key}_rot_blocked"] = got

    # fp32 cases: BASELINE config-4 style inputs at small size
    for idx, (m, n, k, seed) in enumerate([(24, 40, 8, 0), (65, 33, 12, 1)]):
        rng = np.random.Generator(np.random.Philox(seed))
        A32 = np.asfortranarray(rng.uniform(-1.0, 1.0, size=(m, n)).astype(np.float32))
        th = np.random.Generator(np.random.Philox(seed + 1)).uniform(0.0, 2.0 * np.pi, size=(n - 1, k))
        C32 = np.asfortranarray(np.cos(th).astype(np.float32))
        S32 = np.asfortranarray(np.sin(th).astype(np.float32))
        key = f"f{idx}"
        data[f"{key}_A"] = A32
        data[f"{key}_C"] = C32
        data[f"{key}_S"] = S32
        data[f"{key}_rot_right_fwd_f64ref"] = right(A32.astype(np.float64), C32.astype(np.float64),
                                                    S32.astype(np.float64), R, check=False)

    # generate_sequence pin (core.py:94-107)
    g = generate_sequence(10, 4, 1)
    data["gen_C"], data["gen_S"] = g.C, g.S

    # explicit-Q oracle chain (oracle.py:102-136)
    A0, seq = make_inputs(16, 16, 3, 11)
    data["q_A"], data["q_C"], data["q_S"] = A0, seq.C, seq.S
    data["q_Q"] = accumulate_q(seq)
    data["q_AQ"] = reference_multiply(A0, data["q_Q"])

    # non-orthonormal sequence accepted (conftest.py:46-50)
    rng = np.random.Generator(np.random.Philox(0))
    Cn = rng.uniform(-1.2, 1.2, size=(7, 3))
    Sn = rng.uniform(-1.2, 1.2, size=(7, 3))
    rngA = np.random.Generator(np.random.Philox(0))
    An = np.asfortranarray(rngA.standard_normal((9, 8)))
    data["nonorth_A"], data["nonorth_C"], data["nonorth_S"] = An, Cn, Sn
    data["nonorth_out"] = right(An, Cn, Sn, R, check=False)

    np.savez_compressed(OUT, **data)
    print(f"wrote {OUT}: {len(data)} arrays, {os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main()

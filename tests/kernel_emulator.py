"""Numpy emulation of the CUDA band-pipeline arithmetic (test infrastructure).

Restates, index for index, what ``rs_pack_kernel`` and ``run_block`` in
paper_2412_01852_b200/csrc/rotseq_b200.cu compute, vectorised over owners, so the
block / register-slot / coefficient-record algebra can be checked bit for bit
against the oracle on a CPU. Bands are run one after another: the kernel's
ring/flag hand-offs only reorder independent work (checked separately by
pipeline_model), so the arithmetic is the same.
"""

from __future__ import annotations

import numpy as np


def pack(C, S, length, k, K=8, reverse=False, reflector=False):
    """rs_pack_kernel: records [band][b][u][l] (rotation (c, s); reflector (s, d, e));
    idle lanes are zero; reverse mirrors j and negates S (rotation) or C (reflector)."""
    bands = -(-k // K)
    nchunk = (length + K) // (K + 1)
    nblk = nchunk + 1
    width = 3 if reflector else 2
    out = np.zeros((bands, nblk, K + 1, K, width))
    for band in range(bands):
        for b in range(nblk):
            for u in range(K + 1):
                for lane in range(K):
                    p = band * K + lane
                    j = b * (K + 1) + u - 1 - lane
                    if p < k and 0 <= j <= length - 2:
                        jj = length - 2 - j if reverse else j
                        c, s = C[jj, p], S[jj, p]
                        if reflector:
                            if reverse:
                                c = -c
                            out[band, b, u, lane] = (s, c - s, c + s)
                        else:
                            if reverse:
                                s = -s
                            out[band, b, u, lane] = (c, s)
    return out, nblk, nchunk


def _xform(x, y, rec, strict, reflector):
    if reflector:
        s, d, e = rec
        w = s * (x + y)
        return w + d * x, w - e * y  # strict shape; fast mode is not emulated
    c, s = rec
    return c * x + s * y, c * y - s * x


def emulate(A, C, S, side="right", order="forward", kind="rotation", K=8):
    """Apply like the kernel does and return the result (A is not modified)."""
    X = np.array(A, dtype=np.float64, order="F")
    if side == "left":
        X = X.T.copy()  # owners become rows, the rotated dimension columns
    owners, length = X.shape
    if order == "reverse":
        X = X[:, ::-1].copy()  # mirrored column addressing (base + (len-1)*cs, stride -cs)
    k = C.shape[1]
    recs, nblk, nchunk = pack(C, S, length, k, K, order == "reverse", kind == "reflector")
    bands = recs.shape[0]
    for band in range(bands):
        kb = min(K, k - band * K)
        out = np.zeros_like(X)
        w = [np.zeros(owners) for _ in range(K + 1)]
        for b in range(nblk):
            c0 = b * (K + 1)
            for u in range(K + 1):
                if b >= 1:  # emit column (b-1)(K+1)+u from slot u
                    col = c0 - (K + 1) + u
                    if col < length:
                        out[:, col] = w[u]
                col = c0 + u  # load column b(K+1)+u into slot u
                w[u] = X[:, col].copy() if (b < nchunk and col < length) else np.zeros(owners)
                for lane in range(K):
                    sx = (u - 1 - lane) % (K + 1)
                    sy = (sx + 1) % (K + 1)
                    j = c0 + u - 1 - lane
                    if lane >= kb or j < 0 or j > length - 2:
                        continue
                    w[sx], w[sy] = _xform(w[sx], w[sy], recs[band, b, u, lane], True, kind == "reflector")
        X = out
    if order == "reverse":
        X = X[:, ::-1]
    if side == "left":
        X = X.T
    return np.asfortranarray(X)

"""Numpy emulation of the CUDA pipeline arithmetic (test infrastructure).

Restates, index for index, what ``rs_pack_kernel`` / ``rs_pack_scaled_kernel`` and
``run_block`` in paper_2412_01852_b200/csrc/rotseq_b200.cu compute, vectorised over
owners, so the block / register-slot / coefficient-record algebra can be checked on a
CPU. Units (a tile's sweep range of <= K sweeps) run one after another: the kernel's
ring/flag hand-offs only reorder independent work (checked by pipeline_model), so the
arithmetic is the same.

* standard records, strict arithmetic: bit-identical to the oracle;
* scaled ("fast Givens") records: the fast-mode algebra, checked against the oracle
  within the fast-mode tolerance (numpy has no FMA, so not bit-exact with the GPU).
"""

from __future__ import annotations

import numpy as np

K_DEFAULT = 8


def unit_partition(k: int, ut: int):
    """Unit i of a tile covers sweeps [floor(i*k/ut), floor((i+1)*k/ut)) (unit_at)."""
    return [(i * k // ut, (i + 1) * k // ut - i * k // ut) for i in range(ut)]


def geometry(length: int, K: int = K_DEFAULT):
    nchunk = (length + K) // (K + 1)
    return nchunk, nchunk + 1


def _forward_cs(C, S, length, j, p, reverse, reflector):
    jj = length - 2 - j if reverse else j
    c, s = C[jj, p], S[jj, p]
    if reverse:
        if reflector:
            c = -c
        else:
            s = -s
    return c, s


def pack_unit(C, S, length, p0, kb, reverse=False, reflector=False, K=K_DEFAULT):
    """rs_pack_kernel for one unit: records [b][u][l] (rotation (c, s); reflector
    (s, d, e)); slots with j outside [0, len-2] are zero."""
    _, nblk = geometry(length, K)
    width = 3 if reflector else 2
    out = np.zeros((nblk, K + 1, kb, width))
    for b in range(nblk):
        for u in range(K + 1):
            for lane in range(kb):
                j = b * (K + 1) + u - 1 - lane
                if 0 <= j <= length - 2:
                    c, s = _forward_cs(C, S, length, j, p0 + lane, reverse, reflector)
                    out[b, u, lane] = (s, c - s, c + s) if reflector else (c, s)
    return out


def pack_unit_scaled(C, S, length, p0, kb, reverse=False, reflector=False, K=K_DEFAULT):
    """rs_pack_scaled_kernel for one unit: (tau1, -tau2) records [b][u][l], the emission
    scale of every column, and whether any value left the safe range."""
    _, nblk = geometry(length, K)
    taus = np.zeros((nblk, K + 1, kb, 2))
    scale = np.ones(length)
    lo, hi = 2.0 ** -256, 2.0 ** 256
    unsafe = False
    for j in range(length):
        sa = sb = 1.0
        for lane in range(kb):
            p = p0 + lane
            if j >= 1:
                c, s = _forward_cs(C, S, length, j - 1, p, reverse, reflector)
                sa *= -c if reflector else c
            if j <= length - 2:
                c, s = _forward_cs(C, S, length, j, p, reverse, reflector)
                with np.errstate(divide="ignore", invalid="ignore"):
                    t1 = s * sb / (c * sa)
                    t2 = s * sa / (c * sb)
                unsafe |= not (c != 0 and abs(t1) <= hi and abs(t2) <= hi)
                bu = j + 1 + lane
                taus[bu // (K + 1), bu % (K + 1), lane] = (t1, -t2)
                sa *= c
                sb *= -c if reflector else c
                if j + 1 <= length - 2:
                    c, s = _forward_cs(C, S, length, j + 1, p, reverse, reflector)
                    sb *= c
            unsafe |= not (lo <= abs(sa) <= hi and lo <= abs(sb) <= hi)
        scale[j] = sa
    return taus, scale, unsafe


def _xform(x, y, rec, reflector):
    if reflector:
        s, d, e = rec
        w = s * (x + y)
        return w + d * x, w - e * y  # strict shape
    c, s = rec
    return c * x + s * y, c * y - s * x


def _run_unit(X, length, p0, kb, recs, scaled, reflector, K=K_DEFAULT):
    """One unit over all blocks (run_block): returns the emitted matrix."""
    owners = X.shape[0]
    nchunk, nblk = geometry(length, K)
    out = np.zeros_like(X)
    w = [np.zeros(owners) for _ in range(K + 1)]
    if scaled:
        taus, scale = recs
    for b in range(nblk):
        c0 = b * (K + 1)
        for u in range(K + 1):
            if b >= 1:  # emit column (b-1)(K+1)+u from slot u
                col = c0 - (K + 1) + u
                if col < length:
                    out[:, col] = w[u] * scale[col] if scaled else w[u]
            col = c0 + u  # load column b(K+1)+u into slot u
            w[u] = X[:, col].copy() if (b < nchunk and col < length) else np.zeros(owners)
            for lane in range(kb):
                sx = (u - 1 - lane) % (K + 1)
                sy = (sx + 1) % (K + 1)
                j = c0 + u - 1 - lane
                if j < 0 or j > length - 2:
                    continue
                if scaled:
                    t1, nt2 = taus[b, u, lane]
                    x, y = w[sx], w[sy]
                    w[sx], w[sy] = x + t1 * y, y + nt2 * x
                else:
                    w[sx], w[sy] = _xform(w[sx], w[sy], recs[b, u, lane], reflector)
    return out


def emulate(A, C, S, side="right", order="forward", kind="rotation", K=K_DEFAULT, ut=None, scaled=False):
    """Apply like the kernel does (units of the ut-way sweep partition, default the
    narrowest full-width one) and return the result (A is not modified)."""
    X = np.array(A, dtype=np.float64, order="F")
    if side == "left":
        X = X.T.copy()  # owners become rows, the rotated dimension columns
    owners, length = X.shape
    if order == "reverse":
        X = X[:, ::-1].copy()  # mirrored column addressing (base + (len-1)*cs, stride -cs)
    k = C.shape[1]
    ut = ut or -(-k // K)
    rev, refl = order == "reverse", kind == "reflector"
    for p0, kb in unit_partition(k, ut):
        if scaled:
            taus, scale, _ = pack_unit_scaled(C, S, length, p0, kb, rev, refl, K)
            X = _run_unit(X, length, p0, kb, (taus, scale), True, refl, K)
        else:
            X = _run_unit(X, length, p0, kb, pack_unit(C, S, length, p0, kb, rev, refl, K), False, refl, K)
    if order == "reverse":
        X = X[:, ::-1]
    if side == "left":
        X = X.T
    return np.asfortranarray(X)

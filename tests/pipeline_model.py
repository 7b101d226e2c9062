"""CPU model of the CUDA pipeline's work split and hand-off protocol.

Mirrors ``plan_launch`` / ``unit_at`` / ``cta_range`` / ``rs_pipeline_kernel`` in
paper_2412_01852_b200/csrc/rotseq_b200.cu: U units numbered tile-major (tile t holds
ua (+1 for t < t1) units splitting the k sweeps evenly), G CTAs with contiguous unit
ranges (the last partial tile first), positions on warp p % NW in rounds, ring
hand-offs between neighbouring positions of a round, progress flags otherwise.

``simulate`` steps every warp as far as its waits allow (round-robin, one block at a
time) and reports a deadlock if no warp can make progress. It also records the order
of (tile, unit, block) events so the schedule's dependency legality can be checked
against the reference's rule (conftest.py:26-43 ``assert_naive_equivalent_order``).
"""

from __future__ import annotations

from dataclasses import dataclass

FLAG_EVERY = 8  # kFlagEvery in rotseq_b200.cu


@dataclass
class Geometry:
    owners: int
    length: int
    k: int
    K: int = 8
    R: int = 2
    S: int = 2

    @property
    def tiles(self):
        return -(-self.owners // (32 * self.R))

    @property
    def nchunk(self):
        return (self.length + self.K) // (self.K + 1)

    @property
    def nblk(self):
        return self.nchunk + 1


def warp_cap(dtype_bytes: int = 8, refl: bool = False, R: int = 2, K: int = 8, S: int = 2,
             optin: int = 232448, max_warps: int = 16, left: bool = False) -> int:
    """plan_launch()'s shared-memory bound on warps per CTA (a multiple of 4). The right
    side's coefficient buffers hold block pairs (coef_blocks_per_buf)."""
    rec = (4 if refl else 2) * dtype_bytes
    cbuf = max((K + 1) * K * max(rec, 16), ((K + 1) * K + 5) * 16)
    per = 2 * (1 if left else 2) * cbuf + S * (K + 1) * 32 * R * dtype_bytes + (S + 3) * 8
    return min(max_warps, (optin - (S + 3) * 8) // per) & ~3


def equal_chain_plan(g: Geometry, grid: int, cap: int, bestG: int, bestU: int, bestNW: int):
    """plan_launch()'s equal-chain candidate: one round, chains of ut' > ut units of mixed
    widths on more SMs than the aligned plan, wide units mid-period (off = ut' // 2)."""
    if not (bestG < grid and bestU // bestNW == bestG and bestU // g.tiles > bestNW):
        return None
    ut_a = bestU // g.tiles

    def cost(ut, nw, per_smsp):
        cross = (-(-ut // nw) - 1) + (0.5 if ut % nw else 0.0)
        return (g.nblk + 2.2 * (ut - 1) + 9.0 * cross) * per_smsp

    best_c = 0.98 * cost(ut_a, bestNW, (bestNW // 4) * (g.k // ut_a))
    pick = None
    for ut in range(ut_a + 1, min(ut_a + ut_a // 4, g.k) + 1):
        if g.k % ut == 0 or g.k // ut < 2:
            continue
        U = g.tiles * ut
        for nw in range(cap, 7, -4):
            if U % nw:
                continue
            G2 = U // nw
            if G2 > grid or G2 <= bestG or (g.k % ut) * 4 > ut:
                continue
            c = cost(ut, nw, (nw // 4) * (g.k // ut) + 1)
            if c < best_c:
                best_c, pick = c, (G2, U, nw)
    if pick is None:
        return None
    G2, U, nw = pick
    ua = U // g.tiles
    return dict(G=G2, U=U, ua=ua, t1=0, NW=nw, off=best_sweep_offset(ua, nw, g.k))


def best_sweep_offset(ut: int, nw: int, k: int) -> int:
    """The offset whose wide units fall least often on a chain's head, tail or flag hand-off
    units (first / last unit of a CTA's range) over the tiles' phases; smallest on ties."""
    w0 = k // ut
    best = None
    for off in range(ut):
        score = 0
        for t in range(nw):
            phase = (t * ut) % nw
            for i in range(ut):
                if sweep_start(i + 1, ut, k, off) - sweep_start(i, ut, k, off) <= w0:
                    continue
                pos = (phase + i) % nw
                if i == 0 or i == ut - 1 or pos == 0 or pos == nw - 1:
                    score += 1
        if best is None or score < best[0]:
            best = (score, off)
    return best[1]


def plan(g: Geometry, sms: int = 148, cap: int = 16, grid: int | None = None, mode: int = 0,
         equal_chain: bool = True, left: bool = False):
    """plan_launch(): grid, U, ua, t1, NW, off (sweep-split offset)."""
    cap = max(4, cap & ~3)
    G = sms if grid is None else min(grid, sms)
    if mode in (0, 3) and grid is None:
        # aligned plan (plan_launch): uniform widths k/ut, chains filling CTA rounds
        best = None
        ut0 = -(-g.k // g.K)
        for ut in range(ut0, min(2 * ut0, g.k) + 1):
            if g.k % ut:
                continue
            U = g.tiles * ut
            for nw in range(cap, 7, -4):
                if not (ut % nw == 0 or nw % ut == 0) or U % nw:
                    continue
                cr = U // nw
                r = -(-cr // G)
                while r <= 4 and cr % r:
                    r += 1
                if r > 4:
                    continue
                G2 = cr // r
                if G2 * 5 < G * 4:
                    continue
                if best is None or G2 > best[0]:
                    best = (G2, U, nw)
        if best is not None:
            G2, U, nw = best
            eq = equal_chain_plan(g, G, cap, G2, U, nw) if (equal_chain and not left) else None
            if eq is not None:
                return eq
            return dict(G=G2, U=U, ua=U // g.tiles, t1=U % g.tiles, NW=nw, off=0)
    umin = g.tiles * -(-g.k // g.K)
    G = max(1, min(G, -(-umin // 4)))
    q = -(-umin // (4 * G))
    if mode == 0:
        w1 = g.k * g.tiles / (4 * G * q)
        mode = 2 if (q >= 8 or w1 > 7.5) else 1
    U = 4 * G * q if mode == 1 else umin
    U = min(U, g.tiles * g.k)
    nmax = -(-U // G)
    rounds = -(-nmax // cap)
    nw = min(cap, -(-(-(-nmax // rounds)) // 4) * 4)
    return dict(G=G, U=U, ua=U // g.tiles, t1=U % g.tiles, NW=nw, off=0)


def tile_first_unit(t, t1, ua):
    return t * (ua + 1) if t < t1 else t1 * (ua + 1) + (t - t1) * ua


def sweep_start(i, ut, k, off=0):
    return 0 if i <= 0 else k if i >= ut else (i * k + off) // ut


def unit_at(gidx, t1, ua, k, off=0):
    big = t1 * (ua + 1)
    if gidx < big:
        tile, i, ut = gidx // (ua + 1), gidx % (ua + 1), ua + 1
    else:
        r = gidx - big
        tile, i, ut = t1 + r // ua, r % ua, ua
    p0 = sweep_start(i, ut, k, off)
    return tile, p0, sweep_start(i + 1, ut, k, off) - p0


def cta_range(U, c, G, t1, ua, k, off=0):
    g0, g1 = U * c // G, U * (c + 1) // G
    nl = 0
    if g1 > g0:
        tile, p0, kb = unit_at(g1 - 1, t1, ua, k, off)
        if p0 + kb < k:
            f = tile_first_unit(tile, t1, ua)
            if f > g0:
                nl = g1 - f
    return g0, g1, nl


def cta_schedule(g: Geometry, pl: dict, c: int):
    """List of (pos, warp, round, unit gidx, (tile, p0, kb), src, dst) for CTA c."""
    U, G, t1, ua, NW, k = pl["U"], pl["G"], pl["t1"], pl["ua"], pl["NW"], g.k
    off = pl.get("off", 0)
    g0, g1, nl = cta_range(U, c, G, t1, ua, k, off)

    def pos_to_unit(p):
        return g1 - nl + p if p < nl else g0 + p - nl

    def unit_to_pos(u):
        return u - (g1 - nl) if u >= g1 - nl else u - g0 + nl

    out = []
    for p in range(g1 - g0):
        w, jr = p % NW, p // NW
        u = pos_to_unit(p)
        tile, p0, kb = unit_at(u, t1, ua, k, off)
        src = "global"
        if p0 > 0:
            src = "ring" if (w > 0 and u - 1 >= g0 and unit_to_pos(u - 1) == p - 1) else "flag"
        dst = "global"
        if p0 + kb < k:
            dst = "ring" if (w < NW - 1 and u + 1 < g1 and unit_to_pos(u + 1) == p + 1) else "flag"
        out.append((p, w, jr, u, (tile, p0, kb), src, dst))
    return out


def simulate(g: Geometry, sms: int = 148, cap: int = 16, grid: int | None = None, mode: int = 0,
             max_steps: int = 20_000_000):
    pl = plan(g, sms, cap, grid, mode)
    S, nchunk, nblk, NW = g.S, g.nchunk, g.nblk, pl["NW"]
    warps = []
    for c in range(pl["G"]):
        sched = cta_schedule(g, pl, c)
        for w in range(NW):
            warps.append(dict(cta=c, warp=w, work=[e for e in sched if e[1] == w], idx=0, b=-1))
    full, consumed, flags, order = {}, {}, {}, {}
    active = [ws for ws in warps if ws["work"]]
    steps = 0
    while active:
        progressed = False
        for ws in active:
            p, w, jr, u, (tile, p0, kb), src, dst = ws["work"][ws["idx"]]
            seq0 = jr * nchunk
            rin, rout = (ws["cta"], w), (ws["cta"], w + 1)
            myflag, outflag = (tile, p0), (tile, p0 + kb)
            if ws["b"] == -1:  # prologue: self-fill chunk 0
                if src != "ring":
                    if src == "flag" and flags.get(myflag, 0) < 1:
                        continue
                    full[rin] = full.get(rin, 0) + 1
                ws["b"] = 0
                progressed = True
                continue
            b = ws["b"]
            self_fill = src != "ring"
            if self_fill and b + 1 < nchunk and src == "flag" and flags.get(myflag, 0) < b + 2:
                continue
            has_in, has_out = b < nchunk, b >= 1
            iseq, oseq = seq0 + b, seq0 + b - 1
            if has_in and full.get(rin, 0) < iseq + 1:
                continue
            if dst == "ring" and has_out and oseq >= S and consumed.get(rout, 0) < oseq - S + 1:
                continue
            order.setdefault(tile, []).append((p0, kb, b))
            if has_in:
                consumed[rin] = iseq + 1
            if dst == "ring" and has_out:
                full[rout] = full.get(rout, 0) + 1
            if dst == "flag" and has_out and (b < 2 * FLAG_EVERY or b % FLAG_EVERY == 0 or b == nblk - 1):
                flags[outflag] = b
            if self_fill and b + 1 < nchunk:
                full[rin] = full.get(rin, 0) + 1
            ws["b"] += 1
            if ws["b"] >= nblk:
                ws["idx"] += 1
                ws["b"] = -1
            progressed = True
            steps += 1
            if steps > max_steps:
                raise RuntimeError("step limit exceeded")
        active = [ws for ws in active if ws["idx"] < len(ws["work"])]
        if not progressed:
            stuck = [(ws["cta"], ws["warp"], ws["work"][ws["idx"]], ws["b"]) for ws in active][:12]
            raise RuntimeError(f"deadlock: {pl}; stuck warps (cta, warp, work, block): {stuck}")
    return dict(plan=pl, order=order)


def unit_block_rotations(g: Geometry, p0: int, kb: int, b: int):
    """Rotations (j, p) of block b of a unit, in the kernel's order (run_block):
    wave u = 0..K (t = b(K+1)+u-1), lanes l ascending, j = t - l."""
    K = g.K
    for u in range(K + 1):
        t = b * (K + 1) + u - 1
        for lane in range(kb):
            j = t - lane
            if 0 <= j <= g.length - 2:
                yield j, p0 + lane

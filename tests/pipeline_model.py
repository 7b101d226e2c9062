"""CPU model of the CUDA band-pipeline's work split and hand-off protocol.

Mirrors ``rs_pipeline_kernel`` in paper_2412_01852_b200/csrc/rotseq_b200.cu:
unit list split over CTAs, the in-CTA processing order (tail-first reorder),
rounds of NW warps, src/dst selection (ring vs. global vs. progress flag),
ring full/empty barriers with S stages, and per-unit progress flags.

``simulate`` steps every warp as far as its waits allow (round-robin, one block
at a time) and reports a deadlock if no warp can make progress. It also records
the order in which transforms (q, p) are applied to each owner line so the
schedule's dependency legality can be checked against the reference's rule
(conftest.py:26-43 ``assert_naive_equivalent_order``).
"""

from __future__ import annotations

from dataclasses import dataclass, field


FLAG_EVERY = 8  # kFlagEvery in rotseq_b200.cu


@dataclass
class Geometry:
    owners: int
    length: int
    k: int
    K: int = 8
    R: int = 2
    S: int = 3

    @property
    def tile_owners(self):
        return 32 * self.R

    @property
    def bands(self):
        return -(-self.k // self.K)

    @property
    def tiles(self):
        return -(-self.owners // self.tile_owners)

    @property
    def units(self):
        return self.tiles * self.bands

    @property
    def nchunk(self):
        return (self.length + self.K) // (self.K + 1)

    @property
    def nblk(self):
        return self.nchunk + 1


def warp_cap(dtype_bytes: int = 8, refl: bool = False, R: int = 2, K: int = 8, S: int = 3,
             optin: int = 232448, max_warps: int = 16) -> int:
    """plan_launch()'s shared-memory bound on warps per CTA."""
    rec = (4 if refl else 2) * dtype_bytes
    per = 2 * (K + 1) * K * rec + S * (K + 1) * 32 * R * dtype_bytes + (S + 3) * 8
    return min(max_warps, (optin - (S + 3) * 8) // per)


def plan(g: Geometry, sms: int = 148, cap: int = 14, grid: int | None = None):
    """plan_launch(): grid, warps per CTA."""
    import math

    G = min(sms if grid is None else grid, g.units)
    G = max(G, 1)
    x = g.units / G
    rounds = max(1, math.ceil(x / cap))
    nw = min(cap, max(1, math.ceil(x / rounds)))
    return G, nw


def cta_schedule(g: Geometry, G: int, nw: int, c: int):
    """List of (position, warp, round, unit, src, dst) for CTA c."""
    U, bands = g.units, g.bands
    ub, ue = U * c // G, U * (c + 1) // G
    tail_start = (ue // bands) * bands
    reorder = (ue % bands != 0) and tail_start > ub
    ntail = ue - tail_start if reorder else 0

    def unit_at(p):
        return (tail_start + p if p < ntail else ub + (p - ntail)) if reorder else ub + p

    def pos_of(u):
        return ((u - tail_start) if u >= tail_start else (u - ub + ntail)) if reorder else u - ub

    out = []
    for p in range(ue - ub):
        w, jr = p % nw, p // nw
        u = unit_at(p)
        band = u % bands
        if band == 0:
            src = "global"
        elif w > 0 and u - 1 >= ub and pos_of(u - 1) == p - 1:
            src = "ring"
        else:
            src = "flag"
        if band == bands - 1:
            dst = "global"
        elif w < nw - 1 and u + 1 < ue and pos_of(u + 1) == p + 1:
            dst = "ring"
        else:
            dst = "flag"
        out.append((p, w, jr, u, src, dst))
    return out


@dataclass
class WarpState:
    cta: int
    warp: int
    work: list
    idx: int = 0          # index into work
    b: int = -1           # -1: unit prologue pending
    done: bool = False
    cseq: int = 0


@dataclass
class Sim:
    g: Geometry
    G: int
    nw: int
    flags: dict = field(default_factory=dict)
    full: dict = field(default_factory=dict)    # (cta, ring) -> arrivals
    empty: dict = field(default_factory=dict)
    applied: dict = field(default_factory=dict)  # tile -> list of (band, b)


def simulate(g: Geometry, sms: int = 148, cap: int = 14, grid: int | None = None, max_steps: int = 10_000_000):
    G, nw = plan(g, sms, cap, grid)
    sim = Sim(g, G, nw)
    S, nchunk, nblk = g.S, g.nchunk, g.nblk
    warps = []
    for c in range(G):
        sched = cta_schedule(g, G, nw, c)
        for w in range(nw):
            warps.append(WarpState(c, w, [e for e in sched if e[1] == w]))
    arrivals_full = {}
    arrivals_empty = {}
    flags = {}
    order = {}  # tile -> list of band-block events

    def fa(key):
        return arrivals_full.get(key, 0)

    def ea(key):
        return arrivals_empty.get(key, 0)

    steps = 0
    active = [ws for ws in warps if ws.work]
    while active:
        progressed = False
        for ws in active:
            if ws.done:
                continue
            p, w, jr, u, src, dst = ws.work[ws.idx]
            seq0 = jr * nchunk
            ring_in = (ws.cta, w)
            ring_out = (ws.cta, w + 1)
            if ws.b == -1:
                # prologue: self-fill chunk 0
                if src != "ring":
                    if src == "flag" and flags.get(u, 0) < min(2, nchunk):
                        continue
                    arrivals_full[ring_in] = fa(ring_in) + 1
                ws.b = 0
                progressed = True
                continue
            b = ws.b
            self_next = src != "ring" and b + 1 < nchunk
            self_next2 = src != "ring" and b + 2 < nchunk
            if self_next2 and src == "flag" and flags.get(u, 0) < b + 3:
                continue
            has_in, has_out = b < nchunk, b >= 1
            iseq = seq0 + b
            if has_in and fa(ring_in) < iseq + 1:
                continue
            oseq = seq0 + b - 1
            if dst == "ring" and has_out and oseq >= S and ea(ring_out) < oseq - S + 1:
                continue
            # compute block b
            tile, band = divmod(u, g.bands)
            order.setdefault(tile, []).append((band, b))
            if has_in:
                arrivals_empty[ring_in] = ea(ring_in) + 1
            if dst == "ring" and has_out:
                arrivals_full[ring_out] = fa(ring_out) + 1
            if dst == "flag" and has_out and (b % FLAG_EVERY == 0 or b == nblk - 1):
                flags[u + 1] = b
            if self_next:
                arrivals_full[ring_in] = fa(ring_in) + 1
            ws.b += 1
            if ws.b >= nblk:
                ws.idx += 1
                ws.b = -1
                if ws.idx >= len(ws.work):
                    ws.done = True
            progressed = True
            steps += 1
            if steps > max_steps:
                raise RuntimeError("step limit exceeded")
        active = [ws for ws in active if not ws.done]
        if not progressed:
            stuck = [(ws.cta, ws.warp, ws.work[ws.idx], ws.b) for ws in active][:12]
            raise RuntimeError(f"deadlock: G={G} nw={nw}; stuck warps (cta, warp, work, block): {stuck}")
    return dict(G=G, nw=nw, order=order)


def check_band_block_order(g: Geometry, order: dict):
    """Band b+1 block j may only run after band b produced the chunk it reads."""
    for tile, ev in order.items():
        done = {}
        for band, b in ev:
            done[band] = b
            if band > 0 and b < g.nchunk:
                # chunk b of band `band` input = output chunk b of band-1, emitted in its block b+1
                prev = done.get(band - 1, -1)
                assert prev >= min(b + 1, g.nblk - 1), (tile, band, b, prev)


def block_rotations(g: Geometry, band: int, b: int):
    """Rotations (j, p) of block b of a band, in the kernel's order (run_block):
    wave u = 0..K (t = b(K+1)+u-1), lanes l ascending, j = t - l."""
    K = g.K
    kb = min(K, g.k - band * K)
    for u in range(K + 1):
        t = b * (K + 1) + u - 1
        for lane in range(kb):
            j = t - lane
            if 0 <= j <= g.length - 2:
                yield j, band * K + lane

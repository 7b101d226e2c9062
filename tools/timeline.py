"""Timeline analysis of one pipeline launch (needs tools/exp/lib_trace.so, built with -DRS_TRACE)."""
import sys, os
HERE = os.path.dirname(os.path.abspath(__file__))
os.environ.setdefault("RS_LIB_PATH", os.path.join(HERE, "exp", "lib_trace.so"))
sys.path.insert(0, os.path.dirname(HERE))
import numpy as np, torch
from paper_2412_01852_b200 import apply_device, _lib, flops_applied
m, n, k = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (4096, 4096, 192)
side = sys.argv[4] if len(sys.argv) > 4 else "right"
order = sys.argv[5] if len(sys.argv) > 5 else "forward"
ln = m if side == "left" else n
lib = _lib.load()
info = _lib.plan_info(m, n, k, side=1 if side == "left" else 0)
G, NW = info["grid_ctas"], info["warps_per_cta"]
W, RND = 10, 32
buf = torch.zeros(G * 16 * RND * W, dtype=torch.int64, device="cuda")
_lib.check(lib.rs_debug_set_trace(buf.data_ptr()), "trace")
A = torch.randn(n, m, dtype=torch.float64, device="cuda").t()
th = torch.rand(k, ln - 1, dtype=torch.float64, device="cuda").t() * 6.283185307179586
C, S = torch.cos(th), torch.sin(th)
for _ in range(2):
    buf.zero_(); apply_device(A, (C, S), fast=True, side=side, order=order)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
buf.zero_(); e0.record(); apply_device(A, (C, S), fast=True, side=side, order=order); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
rec = buf.cpu().numpy().reshape(G, 16, RND, W)
valid = rec[..., 1] != 0
r = rec[valid]
t0 = r[:, 1].min()
start = (r[:, 1] - t0) / 1e3
end = (r[:, 2] - t0) / 1e3
print(f"{m}x{n} k={k}: {ms:.3f} ms, {flops_applied(m,n,k)/ms/1e9:.2f} TF/s; grid {G} x {NW} warps; units {len(r)}")
print(f"unit duration us: min {np.min(end-start):.1f} med {np.median(end-start):.1f} max {np.max(end-start):.1f}")
print(f"unit start us: min {start.min():.1f} med {np.median(start):.1f} max {start.max():.1f}; end max {end.max():.1f}")
names = ["fill/flag", "coef", "full", "space", "compute", "post"]
tot = r[:, 3:9].sum(axis=0).astype(float)
print("cycle shares:", ", ".join(f"{nm} {100*v/tot.sum():.1f}%" for nm, v in zip(names, tot)))
srcs = (r[:, 0] >> 40) & 0xf
for sv, nm in ((0, "ring"), (1, "global"), (2, "flag")):
    sel = srcs == sv
    if sel.any():
        t = r[sel, 3:9].sum(axis=0).astype(float)
        print(f"  src={nm:6s} n={sel.sum():5d}:", ", ".join(f"{a} {100*v/t.sum():.1f}%" for a, v in zip(names, t)))
nblk = (ln + 8) // 9 + 1
kbs = (r[:, 9] >> 32) & 0xff
per_block_compute = r[:, 7].sum() / (len(r) * nblk)
print("unit widths:", dict(zip(*np.unique(kbs, return_counts=True))))
print(f"compute cycles per warp-block: {per_block_compute:.0f}")
# active units over time (all SMs)
T = end.max(); bins = np.linspace(0, T, 21)
act = [((start < b1) & (end > b0)).sum() for b0, b1 in zip(bins[:-1], bins[1:])]
print("active units per 5% of time:", act)
# per-warp breakdown for a few CTAs
print("per-warp (cta,wid,tile,p0,kb,src,dst): compute% full% space% flag%  total_cycles")
for c in [int(x) for x in os.environ.get("CTAS", "0,1,2,3").split(",")]:
    for w in range(NW):
        x = rec[c, w, 0]
        if x[1] == 0: continue
        u = int(x[0]) & 0xffffffffff; srcv = (int(x[0]) >> 40) & 0xf; dstv = (int(x[0]) >> 44) & 0xf
        p0 = int(x[9]) & 0xffffffff; kb = int(x[9]) >> 32
        cyc = x[3:9].astype(float); tt = cyc.sum()
        print(f"  c{c:3d} w{w:2d} tile {u:5d} p0 {p0:3d} kb {kb} src {['ring','glob','flag'][srcv]} dst {['ring','glob','flag'][dstv]}: "
              f"comp {100*cyc[4]/tt:5.1f} full {100*cyc[2]/tt:5.1f} space {100*cyc[3]/tt:5.1f} flag {100*cyc[0]/tt:5.1f} "
              f"start {(x[1]-t0)/1e3:7.1f} end {(x[2]-t0)/1e3:7.1f} us")

# aggregate per (src,dst) class
import collections
agg = collections.defaultdict(lambda: np.zeros(6))
cnt = collections.Counter()
for rr in r:
    key = (["ring","glob","flag"][(int(rr[0]) >> 40) & 0xf], ["ring","glob","flag"][(int(rr[0]) >> 44) & 0xf])
    agg[key] += rr[3:9]; cnt[key] += 1
for key, v in sorted(agg.items()):
    print(f"  {key[0]:>4s}->{key[1]:<4s} n={cnt[key]:5d}: " + ", ".join(f"{a} {100*x/v.sum():.1f}%" for a, x in zip(names, v)))
if os.environ.get("TRACE_SAVE"):
    np.save(os.environ["TRACE_SAVE"], rec)

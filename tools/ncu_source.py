"""Per-instruction stall analysis of an ncu report (source page, SASS).
Usage: python tools/ncu_source.py REPORT.ncu-rep [top]"""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
H = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
def num(r, k):
    try:
        return float(r[H[k]])
    except (ValueError, KeyError, IndexError):
        return 0.0
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(num(r, "Warp Stall Sampling (All Samples)") for r in data)
print(f"total samples {tot:.0f}")
# by opcode
byop = collections.defaultdict(lambda: [0.0, 0.0, collections.Counter()])
for r in data:
    src = r[H["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    e = byop[op]
    e[0] += num(r, "Warp Stall Sampling (All Samples)")
    e[1] += num(r, "Instructions Executed")
    for k in reasons:
        e[2][k[6:]] += num(r, k)
print("opcode            samples%   inst_executed   top reasons")
for op, (smp, ie, c) in sorted(byop.items(), key=lambda x: -x[1][0])[:25]:
    tr = ", ".join(f"{k} {100*v/tot:.1f}" for k, v in c.most_common(3) if v > 0)
    print(f"{op:16s} {100*smp/tot:6.1f}% {ie:14.0f}   {tr}")
print("\ntop instructions:")
for r in sorted(data, key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))[:top]:
    c = collections.Counter({k[6:]: num(r, k) for k in reasons})
    tr = ", ".join(f"{k} {v:.0f}" for k, v in c.most_common(3) if v > 0)
    print(f"{r[H['Address']]:>8s} {100*num(r,'Warp Stall Sampling (All Samples)')/tot:5.2f}% exec {num(r,'Instructions Executed'):10.0f} {r[H['Source']].strip()[:60]:60s} {tr}")

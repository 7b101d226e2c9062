"""Kernel-only timing (rs_apply_packed between events, back-to-back) of the BASELINE
shapes with device-generated inputs. Usage: python tools/kprobe.py [ENV=VAL,...] ..."""
import sys, os, json, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, os, json
sys.path.insert(0, %r)
import torch
from paper_2412_01852_b200 import PackedSequence, flops_applied, Side, _lib
cases = json.loads(os.environ["CASES"])
out = []
for (m, n, k, dt, side, order) in cases:
    dtype = torch.float64 if dt == "f64" else torch.float32
    A = torch.randn(n, m, dtype=dtype, device="cuda").t()
    ln = m if side == "left" else n
    th = torch.rand(k, ln - 1, dtype=torch.float64, device="cuda").t() * 6.283185307179586
    C, S = torch.cos(th).to(dtype), torch.sin(th).to(dtype)
    ps = PackedSequence((C, S), A.shape, side=side, order=order, dtype=dtype)
    for _ in range(3): ps.apply(A, fast=True)
    torch.cuda.synchronize()
    reps = 10
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): ps.apply(A, fast=True)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    f = flops_applied(m, n, k, Side(side))
    peak = 34.15 if dt == "f64" else 72.4
    out.append("%%s %%dx%%d k=%%d: %%.3f ms %%.2f TF/s (%%.1f%%%%)" %% (dt + "/" + side[0] + "/" + order[0], m, n, k, ms, f / ms / 1e9, 100 * f / ms / 1e9 / peak))
print(os.environ.get("TAG", ""), " | ".join(out), flush=True)
''' % ROOT
CASES = [(4096, 4096, 192, "f64", "right", "forward"), (65536, 2048, 256, "f64", "right", "forward"),
         (8192, 8192, 128, "f32", "right", "forward"), (16384, 16384, 96, "f64", "left", "reverse"),
         (8192, 2048, 256, "f64", "right", "forward")]
if os.environ.get("KP_CASES"):
    CASES = json.loads(os.environ["KP_CASES"])
for tag in (sys.argv[1:] or ["default"]):
    env = dict(os.environ, CASES=json.dumps(CASES), TAG=tag)
    for kv in tag.split(","):
        if "=" in kv:
            k, v = kv.split("=", 1); env[k] = v
    try:
        subprocess.run([sys.executable, "-c", code], env=env, timeout=float(os.environ.get("KP_TIMEOUT", 600)))
    except subprocess.TimeoutExpired:
        print(tag, "TIMEOUT", flush=True)

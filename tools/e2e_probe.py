"""Host<->device copy bandwidth and rs_apply_host timing (developer tool)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2412_01852_b200 import apply_host, make_inputs
m, n, k = 4096, 4096, 192
hA = torch.empty_strided((m, n), (1, m), dtype=torch.float64, pin_memory=True)
hA.normal_()
dA = torch.empty_strided((m, n), (1, m), dtype=torch.float64, device="cuda")
hB = torch.empty_like(hA).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - e0) / reps * 1e3
nb = m * n * 8
print("H2D %.3f ms" % t(lambda: dA.copy_(hA, non_blocking=True)), "(%.1f GB/s)" % (nb / t(lambda: dA.copy_(hA, non_blocking=True)) / 1e6))
print("D2H %.3f ms" % t(lambda: hB.copy_(dA, non_blocking=True)))
def both():
    with torch.cuda.stream(s1): dA.copy_(hA, non_blocking=True)
    with torch.cuda.stream(s2): hB.copy_(dA, non_blocking=True)
print("H2D||D2H %.3f ms" % t(both))
th = np.random.default_rng(0).uniform(0, 2 * np.pi, (n - 1, k))
C, S = np.asfortranarray(np.cos(th)), np.asfortranarray(np.sin(th))
if os.environ.get("PINNED_CS", "1") == "1":
    hC = torch.empty_strided(C.shape, (1, C.shape[0]), dtype=torch.float64, pin_memory=True)
    hS = torch.empty_strided(C.shape, (1, C.shape[0]), dtype=torch.float64, pin_memory=True)
    hC.copy_(torch.from_numpy(C)); hS.copy_(torch.from_numpy(S))
    C, S = hC, hS
for ch in ("16", "32", "64"):
    os.environ["RS_HOST_CHUNKS"] = ch
    print("apply_host chunks", ch, "%.3f ms" % t(lambda: apply_host(hA, (C, S), fast=True), 5))
os.environ["RS_HOST_DEBUG"] = "1"; os.environ["RS_HOST_CHUNKS"] = os.environ.get("DBG_CHUNKS", "16")
apply_host(hA, (C, S), fast=True); torch.cuda.synchronize()
# copies concurrent with the resident pipeline kernel
from paper_2412_01852_b200 import PackedSequence
dB = torch.empty_strided((m, n), (1, m), dtype=torch.float64, device="cuda"); dB.normal_()
dC = torch.from_numpy(np.asfortranarray(np.cos(th))).cuda(); dS = torch.from_numpy(np.asfortranarray(np.sin(th))).cuda()
ps = PackedSequence((dC, dS), (m, n), dtype=torch.float64)
s3 = torch.cuda.Stream()
def with_kernel():
    with torch.cuda.stream(s3): ps.apply(dB, fast=True)
    both()
print("H2D||D2H||kernel %.3f ms" % t(with_kernel))
def kern_only():
    with torch.cuda.stream(s3): ps.apply(dB, fast=True)
print("kernel alone %.3f ms" % t(kern_only))
def both_same():
    with torch.cuda.stream(s1): dA.copy_(hA, non_blocking=True)
    with torch.cuda.stream(s2): hA.copy_(dB, non_blocking=True)
print("H2D||D2H same host buffer %.3f ms" % t(both_same))
half = m * n // 2
hAf = torch.as_strided(hA, (m * n,), (1,)); dAf = torch.as_strided(dA, (m * n,), (1,)); dBf = torch.as_strided(dB, (m * n,), (1,))
def both_halves():
    with torch.cuda.stream(s1): dAf[:half].copy_(hAf[:half], non_blocking=True)
    with torch.cuda.stream(s2): hAf[half:].copy_(dBf[half:], non_blocking=True)
print("H2D(1st half)||D2H(2nd half) same buffer %.3f ms" % t(both_halves))
def both_chunked(nc=32):
    step = m * n // nc
    for i in range(nc):
        with torch.cuda.stream(s1): dAf[i*step:(i+1)*step].copy_(hAf[i*step:(i+1)*step], non_blocking=True)
        with torch.cuda.stream(s2): hBf[i*step:(i+1)*step].copy_(dBf[i*step:(i+1)*step], non_blocking=True)
hBf = torch.as_strided(hB, (m * n,), (1,))
for nc in (8, 32, 64):
    print("H2D||D2H chunked %d: %.3f ms" % (nc, t(lambda: both_chunked(nc))))

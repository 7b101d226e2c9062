import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2412_01852_b200 import apply_host, make_inputs
from oracle import oracle
A0, seq = make_inputs(300, 257, 24, 1)
ref = A0.copy(order="F"); oracle.apply_naive(ref, seq.C, seq.S)
got = A0.copy(order="F")
try:
    apply_host(got, seq)
    print("maxdiff", np.abs(got-ref).max())
except Exception as e:
    print("ERR", e)

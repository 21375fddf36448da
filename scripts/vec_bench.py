"""HBM throughput of the vector kernels at full size (debug entry
mr_debug_vector_bench).  Usage: python scripts/vec_bench.py [CONFIG] [N]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np

import paper_2211_03293_b200 as P

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
ctx = P.Context(0)
cfg, _ = P.setup_workload(ctx, name, n=n, make_state=False)
f = P.lib().mr_debug_vector_bench
f.restype = C.c_int
f.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_int]
out = np.zeros(64)
k = f(ctx.h, out.ctypes.data_as(C.POINTER(C.c_double)), 32)
names = ["update nref=1", "update nref=3", "sum_rhs (3 operands)", "lap7 f_I eval",
         "lap7 Newton residual", "lap7 CG matvec", "cg_update", "cg_p", "recover_fi",
         "reduce wrms", "reduce dot", "reduce max"]
print(f"{name} {cfg['n']}^3 x {cfg['S'] + 1} comps ({ctx.dof * 8 / 1e9:.2f} GB per vector)")
for i in range(k):
    print(f"  {names[i]:22s} {out[2 * i]:8.3f} ms  {out[2 * i + 1]:7.0f} GB/s  {out[2 * i + 1] / 6554.9 * 100:5.1f}%")

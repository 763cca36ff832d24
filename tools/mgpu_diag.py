import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import Csr, Restatement
from paper_1501_00324_b200 import capi, workloads as W
print("CDMC", os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS"), flush=True)
n, _, ro, ci, v = W.elasticity_box(14, 13, 12)
m = Csr.make(n, n, ro, ci, v)
R = Restatement()
b = R.spmv_csr(m, np.ones(n)); diag = R.extract_diagonal(m)
for G in (2, 3, 4):
    mg = capi.Mgpu(m, G, devices=[0] * G)
    for what in ("spmv", "cg"):
        t = time.time()
        try:
            if what == "spmv":
                mg.spmv(np.ones(n))
            else:
                r = mg.cg_solve(b, diag, tol=1e-10, max_iterations=2000)
            print(G, what, "ok", f"{time.time()-t:.2f}s", flush=True)
        except Exception as e:
            print(G, what, "FAIL", e, f"{time.time()-t:.2f}s", flush=True)

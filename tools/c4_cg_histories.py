"""Config-4 Jacobi PCG residual histories on the GPU (k1rs in both row
orders, forced 1000 iterations and tol 1e-8), saved for comparison with the
reference's (tests/golden/c4_cg_*.npz)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import Csr, Restatement
from paper_1501_00324_b200 import capi, workloads as W

n, _, ro, ci, v = W.ventricle_box(170, 170, 170)
m = Csr.make(n, n, ro, ci, v)
b = Restatement().spmv_csr(m, np.ones(n))
a = capi.Csr(n, n, ro, ci, v)
diag = a.extract_diagonal()
out = {}
for order in ("reference", "locality"):
    k = capi.Kernel("k1rs", a, row_order=order)
    for tag, tol, mx in (("forced", 1e-300, 1000), ("tol", 1e-8, 5000)):
        t = time.time()
        r = k.cg_solve(b, diag, tol=tol, max_iterations=mx, permuted=True)
        print(order, tag, r.iterations, r.spmv_calls, r.converged, f"{time.time()-t:.2f}s", flush=True)
        out[f"{order}_{tag}_hist"] = r.residual_history
        out[f"{order}_{tag}_meta"] = np.array([r.iterations, r.spmv_calls, int(r.converged)])
        idx = np.linspace(0, n - 1, 257).astype(np.int64)
        out[f"{order}_{tag}_xs"] = r.solution[idx]
        out[f"{order}_{tag}_xnorm"] = np.array([np.linalg.norm(r.solution)])
os.makedirs("gpurun_out", exist_ok=True)
np.savez_compressed("gpurun_out/c4_gpu_histories.npz", **out)

import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import Csr, Restatement
from paper_1501_00324_b200 import capi, workloads as W
R = Restatement()
n, _, ro, ci, v = W.elasticity_box(40, 40, 40)
m = Csr.make(n, n, ro, ci, v)
b = R.spmv_csr(m, np.ones(n)); diag = R.extract_diagonal(m)
th = os.cpu_count()
lay = R.build_k1(m); ref = R.cg_layout(lay, b, diag=diag, tol=1e-300, max_iterations=400, threads=th); R.free(lay)
op, _ = R.reorder(m, True); lay = R.build_k1(op)
perm = R.cg_layout(lay, b, diag=diag, permuted=True, tol=1e-300, max_iterations=400, threads=th); R.free(lay)
hk = ref.residual_history
def fc(h, thr):
    d = np.abs(h - hk) / (1 + hk); i = np.flatnonzero(d > thr); return (int(i[0]) if i.size else None, float(d.max()))
a = capi.Csr(n, n, ro, ci, v)
runs = {"ref-k1rs": perm.residual_history}
runs["gpu-k1"] = capi.Kernel("k1", a).cg_solve(b, diag, tol=1e-300, max_iterations=400).residual_history
runs["gpu-k1rs"] = capi.Kernel("k1rs", a).cg_solve(b, diag, tol=1e-300, max_iterations=400, permuted=True).residual_history
for G in (1, 2, 4):
    runs[f"dist{G}-copy"] = capi.Dist.local(m, G, transport="copy").cg_solve(b, diag, tol=1e-300, max_iterations=400).residual_history
for k, h in runs.items():
    print(k, [fc(h, t) for t in (1e-12, 1e-11, 1e-10)], flush=True)
print("hist", hk[[0, 50, 100, 200, 300, 400]])

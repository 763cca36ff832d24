"""Protocol overhead of the partitioned CG measured on ONE GPU: config-2's
operator in G = 1, 2, 4, 8 blocks (ew_mgpu_*, every block on device 0, one
host thread and stream each; and the in-process peer transport, one stream).
Total work is the same; the difference per iteration is what the halo
exchange and the rank-ordered reductions add (here serialised on one GPU,
so an upper bound of what they add on G GPUs)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import Csr
from paper_1501_00324_b200 import capi, workloads as W

n, _, ro, ci, v = W.elasticity_box(86, 86, 86)
m = Csr.make(n, n, ro, ci, v)
a = capi.Csr(n, n, ro, ci, v)
b = a.spmv(np.ones(n)); diag = a.extract_diagonal()
its = 500
k = capi.Kernel("k1", a)
for _ in range(2): k.cg_solve(b, diag, tol=1e-300, max_iterations=its)
t = time.perf_counter(); k.cg_solve(b, diag, tol=1e-300, max_iterations=its); t1 = time.perf_counter() - t
print(f"single kernel: {t1 / its * 1e6:.1f} us/it", flush=True)
for G in (1, 2, 4, 8):
    for kind in ("mgpu", "peer"):
        if kind == "peer" and G == 1:
            continue
        d = capi.Mgpu(m, G, devices=[0] * G) if kind == "mgpu" else capi.Dist.local(m, G, transport="peer")
        for _ in range(2): d.cg_solve(b, diag, tol=1e-300, max_iterations=its)
        t = time.perf_counter(); r = d.cg_solve(b, diag, tol=1e-300, max_iterations=its); dt = time.perf_counter() - t
        assert r.iterations == its
        print(f"{kind} G={G}: {dt / its * 1e6:.1f} us/it", flush=True)
        del d

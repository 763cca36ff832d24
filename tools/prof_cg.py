"""Kernel timeline of CG iterations (torch profiler / CUPTI): per-kernel
durations and the gaps between them, averaged over the iterations of one
solve. argv: config (c4 | c2), row order, iterations."""
import json, os, sys
from collections import defaultdict
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1501_00324_b200 import capi, workloads as W

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c4"
order = sys.argv[2] if len(sys.argv) > 2 else "locality"
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 200
if cfgname == "c4":
    n, _, ro, ci, v = W.ventricle_box(170, 170, 170); kid = "k1rs"
else:
    n, _, ro, ci, v = W.elasticity_box(86, 86, 86); kid = "k1"
a = capi.Csr(n, n, ro, ci, v)
k = capi.Kernel(kid, a, row_order=order if kid == "k1rs" else "reference")
perm = kid == "k1rs"
b = torch.tensor(a.spmv(np.ones(n)), device="cuda"); d = torch.tensor(a.extract_diagonal(), device="cuda")
for _ in range(3):
    k.cg_solve(b, d, tol=1e-300, max_iterations=iters, permuted=perm)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    k.cg_solve(b, d, tol=1e-300, max_iterations=iters, permuted=perm)
    torch.cuda.synchronize()
prof.export_chrome_trace("/tmp/cg_trace.json")
ev = [e for e in json.load(open("/tmp/cg_trace.json"))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
dur = defaultdict(list); gap = defaultdict(list)
for prev, e in zip(ev, ev[1:]):
    nm = e["name"].split("(")[0][-40:]
    dur[nm].append(e["dur"]); gap[nm].append(e["ts"] - (prev["ts"] + prev["dur"]))
span = (ev[-1]["ts"] + ev[-1]["dur"] - ev[0]["ts"])
print(f"{cfgname} {order}: {len(ev)} events, {span:.0f} us for {iters} iterations = {span/iters:.2f} us/it")
for nm in dur:
    print(f"{len(dur[nm]):6d} x {np.mean(dur[nm]):8.2f} us  gap before {np.median(gap[nm]):6.2f} us  {nm}")

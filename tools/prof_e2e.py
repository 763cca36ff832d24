"""Timeline of host-buffer ew_kernel_apply calls (config 2, K1) via the
torch profiler's CUPTI activity trace: kernels and copies with start/end."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1501_00324_b200 import capi, workloads as W
if os.environ.get("EW_AB_LIB"):  # A/B: another build of the library
    capi.LIB_PATH = os.environ["EW_AB_LIB"]

dims = tuple(int(a) for a in (sys.argv[1] if len(sys.argv) > 1 else "86,86,86").split(","))
n, nc, ro, ci, v = W.elasticity_box(*dims)
a = capi.Csr(n, nc, ro, ci, v)
k = capi.Kernel("k1", a)
x = torch.empty(nc, dtype=torch.float64, pin_memory=True); x.copy_(torch.rand(nc, dtype=torch.float64))
y = torch.empty(n, dtype=torch.float64, pin_memory=True)
xn, yn = x.numpy(), y.numpy()
if os.environ.get("EW_SOAK"):
    xd = torch.tensor(xn, device="cuda"); yd = torch.empty(n, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream()
    t = time.perf_counter()
    while time.perf_counter() - t < float(os.environ["EW_SOAK"]):
        for _ in range(50): k.apply(xd, yd, stream=st)
        torch.cuda.synchronize()
for _ in range(5): k.apply(xn, yn)
for rep in range(3):
    t = time.perf_counter()
    for _ in range(200): k.apply(xn, yn)
    print("ms/call", (time.perf_counter() - t) / 200 * 1e3, flush=True)
if os.environ.get("EW_NO_TRACE"):
    sys.exit(0)
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(3): k.apply(xn, yn)
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace("gpurun_out/e2e_trace.json")
ev = json.load(open("gpurun_out/e2e_trace.json"))["traceEvents"]
g = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
g.sort(key=lambda e: e["ts"])
t0 = g[0]["ts"]
for e in g:
    print(f'{e["ts"]-t0:9.1f} {e["dur"]:8.1f} s{e.get("args",{}).get("stream")} {e["name"][:70]}')

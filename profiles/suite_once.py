"""One launch of every kernel id (K2 at thresholds 4 / 8 / 16) on each of the
config-3 matrices (Table 2 stand-ins), for an ncu launch list
(profiles/capture.sh). argv[1] (optional): comma-separated matrix names."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1501_00324_b200 import capi, load_ellwarp, workloads as W  # noqa: E402

ew_mod = load_ellwarp()
only = set(sys.argv[1].split(",")) if len(sys.argv) > 1 and sys.argv[1] else None
kids = sys.argv[2].split(",") if len(sys.argv) > 2 else ["k1", "k1rs", "k2:4", "k2:8", "k2:16", "csr_vector", "hyb"]
for name, *_ in W.TABLE2:
    if only and name not in only:
        continue
    n, nc, ro, ci, v = W.table2_matrix(name, ew_mod)
    a = capi.Csr(n, nc, ro, ci, v)
    x = torch.tensor(np.random.default_rng(1).uniform(0.1, 1.0, nc), device="cuda")
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    for spec in kids:
        kid, _, th = spec.partition(":")
        try:
            k = capi.Kernel(kid, a, threshold=int(th or 0))
        except capi.DeviceError:
            continue
        (k.apply_permuted if k.has_perm else k.apply)(x, y)
        torch.cuda.synchronize()
        print(name, kid, th, flush=True)
    del a
    torch.cuda.empty_cache()

"""One launch of every kernel id (K2 at its bench-best threshold) on each of
the config-3 structures, for an ncu launch list (profiles/capture.sh)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1501_00324_b200 import capi, load_ellwarp  # noqa: E402

ew_mod = load_ellwarp()
for name, n, kind, p in bench.SUITE:
    m = bench.suite_matrix(ew_mod, kind, n, p)
    a = capi.Csr(m.nrows, m.ncols, np.asarray(m.row_offsets, np.int64), np.asarray(m.col_indices, np.int64),
                 np.asarray(m.values))
    x = torch.tensor(np.random.default_rng(1).uniform(0.1, 1.0, m.ncols), device="cuda")
    y = torch.empty(m.nrows, dtype=torch.float64, device="cuda")
    for kid, th in (("k1", 0), ("k1rs", 0), ("k2", 4), ("k2", 8), ("csr_vector", 0), ("hyb", 0)):
        try:
            k = capi.Kernel(kid, a, threshold=th)
        except capi.DeviceError:
            continue
        (k.apply_permuted if k.has_perm else k.apply)(x, y)
        torch.cuda.synchronize()
        print(name, kid, th, flush=True)
    del a
    torch.cuda.empty_cache()

"""Column span per layout warp of config 4's k1rs operand in the locality
row order (how many warps would take 16-bit column offsets)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1501_00324_b200 import capi, workloads as W

n, _, ro, ci, v = W.ventricle_box(170, 170, 170)
a = capi.Csr(n, n, ro, ci, v)
for order in ("locality", "reference"):
    k = capi.Kernel("k1rs", a, row_order=order)
    fwd, inv = k.perm()
    info = k.info()
    rows = np.repeat(np.arange(n), np.diff(ro))
    w = inv[rows] // 32
    c = inv[ci]
    nw = (n + 31) // 32
    lo = np.full(nw, np.iinfo(np.int64).max); hi = np.full(nw, -1)
    np.minimum.at(lo, w, c); np.maximum.at(hi, w, c)
    span = hi - lo
    slots = np.bincount(w, minlength=nw)
    print(order, "narrow_slots", info.narrow_slots, "stored", info.stored_slots,
          "warps<=65534:", float(np.mean(span <= 65534)), "slot share", float(slots[span <= 65534].sum() / slots.sum()),
          "span pct 50/90/99/max", np.percentile(span, [50, 90, 99]).tolist(), int(span.max()), flush=True)

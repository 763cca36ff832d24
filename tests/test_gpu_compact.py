"""K1 layouts with 16-bit column offsets (compact_layout in ew_layout.cu).

Layouts whose slabs stream from HBM (values + columns over 64 MB) keep, per
layout warp whose real columns lie within 0xFFFF of each other, 16-bit
offsets from the warp's smallest column; other warps stay on the int32 slab.
Same lane sums, so the kernels stay bitwise equal to the reference K1
(warp_spmv.cpp:9-60). These matrices are sized just past the 64 MB gate and
mix narrow warps, wide warps (random columns) and padded warps (row-length
class changes)."""
import numpy as np
import pytest

from oracle.oracle import Csr
from tests.gpu_helpers import bits, oracle_apply, rel_close
from tests.test_gpu_cg import assert_history

pytestmark = pytest.mark.gpu


def mixed(n=1_200_000, seed=7):
    """Row r: length 4 + (r // 50000) % 9; runs of length 12 get columns
    spread over the whole range (wide warps), the rest r + 37 j (mod n)
    (narrow warps, whatever the row numbering the r / rs ids sort into),
    one run three clusters 40,000 apart (wide).
    Length classes recur every 9 runs, so warps at the joints span far (wide)
    or mix lengths (padding)."""
    rng = np.random.default_rng(seed)
    r = np.arange(n, dtype=np.int64)
    lens = 4 + (r // 50000) % 9
    rows = np.repeat(r, lens)
    ro = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=ro[1:])
    j = np.arange(rows.size) - np.repeat(ro[:-1], lens)
    base = np.repeat(np.where(lens == 12, rng.integers(0, n, n), r), lens)
    step = np.where(np.repeat(lens == 12, lens), 104729, 37)  # distinct columns per row
    cols = (base + j * step) % n
    # rows 350,000-399,999: three clusters 40,000 columns apart
    three = np.repeat(r // 50000 == 7, lens)  # one run of them
    cols = np.where(three, (rows + (j % 3 - 1) * 40000 + 37 * (j // 3)) % n, cols)
    cols = np.sort(rows * n + cols) - rows * n  # ascending within each row
    vals = rng.uniform(0.1, 1.0, rows.size)
    return Csr.make(n, n, ro, cols, vals)


@pytest.fixture(scope="module")
def mx():
    return mixed()


def dev(ew, m):
    return ew.Csr(m.nrows, m.ncols, m.row_offsets, m.col_indices, m.values)


def compact_in_use(k):
    """Most slots stream 16-bit columns (ew_kernel_info.narrow_slots), and
    the layout holds no int32 columns for them (shrink_columns: 8 B of value
    + 2 B of offset per narrow slot, int32 only for the wide warps)."""
    i = k.info()
    return (i.narrow_slots * 2 > i.stored_slots and i.device_bytes >= 10 * i.narrow_slots
            and i.col_stream_bytes == 2 * i.narrow_slots + 4 * (i.stored_slots - i.narrow_slots)
            and i.device_bytes < 12 * i.stored_slots + 40 * i.nrows)


@pytest.mark.parametrize("kid", ["k1", "k1r", "k1rs"])
def test_mixed_spans_bitwise(ew, R, mx, kid):
    a = dev(ew, mx)
    x = np.random.default_rng(11).uniform(0.1, 1.0, mx.ncols)
    k = ew.Kernel(kid, a)
    assert k.stored_slots * 12 > 64 << 20
    assert compact_in_use(k), kid
    y = k.apply(x)
    assert np.array_equal(bits(y), bits(oracle_apply(R, kid, mx, x))), kid
    assert rel_close(y, R.spmv_csr(mx, x), 1e-12)
    if k.has_perm:
        fwd, inv = k.perm()
        assert np.array_equal(bits(k.apply_permuted(x[fwd])[inv]), bits(y))


def test_mixed_spans_refresh(ew, R, mx):
    """Values-only refresh keeps the 16-bit columns valid."""
    a = dev(ew, mx)
    k = ew.Kernel("k1", a)
    v2 = mx.values * 3.0 - 0.5
    m2 = Csr.make(mx.nrows, mx.ncols, mx.row_offsets, mx.col_indices, v2)
    k.refresh_values(dev(ew, m2))
    x = np.random.default_rng(12).uniform(-1.0, 1.0, mx.ncols)
    assert np.array_equal(bits(k.apply(x)), bits(oracle_apply(R, "k1", m2, x)))


def test_laplacian_cg_compact(ew, R, F):
    """Jacobi PCG on a 7-point Laplacian past the gate: the fused p.q SpMV on
    the compact slab, history within the reference comparator (k1rs moves
    the boundary rows behind the interior ones: its warps reach further)."""
    m = F.laplacian3d(100, 100, 100)
    b = R.spmv_csr(m, np.ones(m.ncols))
    a = dev(ew, m)
    diag = a.extract_diagonal()
    ref = R.cg_csr(m, b, max_iterations=150)
    for kid in ("k1", "k1rs"):
        k = ew.Kernel(kid, a)
        if kid == "k1":
            assert compact_in_use(k)
        res = k.cg_solve(b, diag, max_iterations=150)
        assert res.iterations == ref.iterations
        assert_history(res.residual_history, ref.residual_history)


_CORPUS_SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, {root!r})
from oracle.oracle import Reference, Restatement
from paper_1501_00324_b200 import capi as ew
from tests.gpu_helpers import bits, oracle_apply
R, F = Restatement(), Reference()
narrow = 0
for case in range(0, 40, 2):
    m = F.random_case(case)
    x = F.random_vector(m.ncols, 7000 + case)
    a = ew.Csr(m.nrows, m.ncols, m.row_offsets, m.col_indices, m.values)
    for ws in (4, 8, 32):
        for kid in ("k1", "k1r", "k1rs"):
            if kid != "k1" and m.nrows != m.ncols:
                continue
            k = ew.Kernel(kid, a, warp_size=ws)
            narrow += k.info().narrow_slots
            y = k.apply(x)
            assert np.array_equal(bits(y), bits(oracle_apply(R, kid, m, x, ws))), (case, kid, ws)
assert narrow > 0
# fused p.q SpMV on compact layouts: CG on the reference's SPD family
for n in (6, 10):
    m = F.laplacian3d(n, n, n)
    b = R.spmv_csr(m, np.ones(m.ncols))
    ref = R.cg_csr(m, b)
    a = ew.Csr(m.nrows, m.ncols, m.row_offsets, m.col_indices, m.values)
    for kid in ("k1", "k1rs"):
        k = ew.Kernel(kid, a)
        res = k.cg_solve(b, a.extract_diagonal())
        assert res.converged and res.iterations == ref.iterations, (n, kid)
        assert np.all(np.abs(res.residual_history - ref.residual_history) <= 1e-10 * (1 + ref.residual_history))
print("ok", narrow)
"""


def test_compact_at_any_size_corpus(ew, F):
    """EW_COMPACT=2 (16-bit columns at any size, a test-only setting) over the
    reference's random corpus at warp sizes 4, 8, 32: every K1 id bitwise
    against the restated reference, and CG histories on compact layouts."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, EW_COMPACT="2")
    out = subprocess.run([sys.executable, "-c", _CORPUS_SCRIPT.format(root=root)], env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    assert out.stdout.strip().startswith("ok")

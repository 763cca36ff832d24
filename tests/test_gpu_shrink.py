"""K1 layouts whose kernels read 16-bit or grouped column lists drop the
int32 column slab (shrink_columns, ew_layout.cu): a compact layout keeps
int32 columns for its wide warps only, a grouped int32 one none. The
layout still exports the reference's arrays (columns decoded from the
kept forms), and every path that read the slab gives the same bits: the
SpMV ids, the host-buffer pipeline's plan, a partition's boundary rows
(split-x K1, restore_columns), the CG."""
import numpy as np
import pytest

from oracle.oracle import Csr
from tests.gpu_helpers import bits, oracle_apply

pytestmark = pytest.mark.gpu

K1_FIELDS = ("values", "col_indices", "warp_offset", "maxrows", "rows_in_warp", "forward", "sorted_row_length")


@pytest.fixture(scope="module")
def elast():
    """3-DOF elasticity box: 206k rows, ~16M nnz -- a slab over 64 MB
    (compact) whose node triples share column lists (grouped)."""
    from paper_1501_00324_b200 import workloads as W

    n, _, ro, ci, v = W.elasticity_box(40, 40, 40)
    return Csr.make(n, n, ro, ci, v)


def dev(ew, m):
    return ew.Csr(m.nrows, m.ncols, m.row_offsets, m.col_indices, m.values)


def test_layout_without_int32_columns_exports_reference_arrays(ew, R, elast):
    a = dev(ew, elast)
    lay = ew.Layout.build(a, "k1")
    i = lay.info()
    assert i.narrow_slots > 0.9 * i.stored_slots  # 16-bit offsets
    assert i.col_stream_bytes < 2 * i.stored_slots  # grouped lists
    assert i.device_bytes < 11.5 * i.stored_slots  # values + the kept column forms, no int32 slab
    got = lay.export()
    want = R.build_k1(elast)
    for f in K1_FIELDS:
        assert np.array_equal(getattr(got, f), getattr(want, f)), f
    R.free(want)


@pytest.mark.parametrize("kid", ["k1", "k1r", "k1rs"])
def test_spmv_ids_bitwise(ew, R, elast, kid):
    a = dev(ew, elast)
    x = np.random.default_rng(3).uniform(-1, 1, elast.ncols)
    k = ew.Kernel(kid, a)
    assert np.array_equal(bits(k.apply(x)), bits(oracle_apply(R, kid, elast, x)))
    x[0] = np.inf  # padding terms 0 * x[0]
    assert np.array_equal(bits(k.apply(x)), bits(oracle_apply(R, kid, elast, x)))


def test_host_buffer_pipeline_bitwise(ew, R, elast):
    """ew_kernel_apply with host buffers (>= 2M nnz: the staged pipeline,
    whose plan reads every slot's column) on the shrunk layout."""
    a = dev(ew, elast)
    k = ew.Kernel("k1", a)
    x = np.random.default_rng(4).uniform(-1, 1, elast.ncols)
    want = oracle_apply(R, "k1", elast, x)
    for _ in range(2):
        assert np.array_equal(bits(k.apply(x)), bits(want))


def test_partition_boundary_rows_bitwise(ew, elast):
    """Two partitions in process: interior rows on the shrunk layout, the
    boundary rows' split-x K1 on a restored int32 slab -- the single-GPU K1
    bits."""
    a = dev(ew, elast)
    x = np.random.default_rng(5).uniform(-1, 1, elast.ncols)
    single = ew.Kernel("k1", a).apply(x)
    d = ew.Dist.local(elast, 2, transport="peer")
    y = d.spmv(x)
    assert np.array_equal(bits(y), bits(single))


def test_cg_on_shrunk_layout(ew, R, elast):
    """The CG's fused SpMV + p.q on the shrunk layout: the reference CG's
    residual history within the reference comparator (test_solver.cpp:
    104-112) over 100 forced iterations."""
    a = dev(ew, elast)
    k = ew.Kernel("k1", a)
    b = R.spmv_csr(elast, np.ones(elast.ncols))
    diag = R.extract_diagonal(elast)
    res = k.cg_solve(b, diag, tol=1e-300, max_iterations=100)
    ref = R.cg_csr(elast, b, tol=1e-300, max_iterations=100)
    assert res.iterations == 100
    dev_ = np.abs(res.residual_history - ref.residual_history) / (1 + ref.residual_history)
    assert np.all(dev_ <= 1e-10)


@pytest.mark.parametrize("kid", ["k1", "k1rs"])
def test_values_refresh_on_shrunk_layout(ew, R, elast, kid):
    """Values-only refresh (the FEM Newton loop's path) on a layout without
    its int32 slab: the kept column forms stay valid, the SpMV is the
    reference's on the new values, host-buffer pipeline included."""
    a = dev(ew, elast)
    k = ew.Kernel(kid, a)
    v2 = elast.values * 3.0 - 0.5
    m2 = Csr.make(elast.nrows, elast.ncols, elast.row_offsets, elast.col_indices, v2)
    k.refresh_values(dev(ew, m2))
    x = np.random.default_rng(13).uniform(-1.0, 1.0, elast.ncols)
    assert np.array_equal(bits(k.apply(x)), bits(oracle_apply(R, kid, m2, x)))

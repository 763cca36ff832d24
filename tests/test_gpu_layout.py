"""Device format construction parity: sort_rows_desc, build_k1 / build_k2,
value_slot_map, make_reordered_r/rs, dump_layout -- every array bit-exact
against the restated oracle and the reference goldens
(test_ellwarp.cpp:40-273, 413-447)."""
import numpy as np
import pytest

from oracle.oracle import Csr

pytestmark = pytest.mark.gpu

K1_FIELDS = ("values", "col_indices", "warp_offset", "maxrows", "rows_in_warp", "forward",
             "sorted_row_length")
K2_FIELDS = K1_FIELDS + ("reduction", "rows_offset_warp")


def dev_csr(ew, m):
    return ew.Csr(m.nrows, m.ncols, m.row_offsets, m.col_indices, m.values)


def _m(d):
    return Csr.make(d["nrows"], d["ncols"], d["row_offsets"], d["col_indices"], d["values"])


def assert_layout_equal(got, want, fields):
    for f in fields:
        a, b = getattr(got, f), getattr(want, f)
        assert a.shape == b.shape and np.array_equal(a, b), f
    assert got.stored_slots == want.stored_slots


def test_goldens(ew, golden):
    a = dev_csr(ew, _m(golden["worked"]["matrix"]))
    fwd, inv = a.sort_rows_desc()
    assert fwd.tolist() == [1, 4, 6, 2, 0, 3, 5]
    r, f2 = a.reorder(False)
    assert f2.tolist() == fwd.tolist()
    assert r.export()[1][:5].tolist() == [4, 0, 5, 1, 6]
    rs, _ = a.reorder(True)
    _, ci, v = rs.export()
    assert ci[:5].tolist() == [0, 1, 4, 5, 6] and v[:5].tolist() == [8.0, 10.0, 7.0, 9.0, 2.0]
    assert dev_csr(ew, _m(golden["sort_132"]["matrix"])).sort_rows_desc()[0].tolist() == [1, 2, 0]
    lay = ew.Layout.build(dev_csr(ew, _m(golden["k1_four_rows"]["matrix"])), "k1", warp_size=4).export()
    assert lay.maxrows.tolist() == [4] and lay.stored_slots == 16 and lay.padded_slots == 6
    g = golden["dump"]
    d = dev_csr(ew, _m(g["matrix"]))
    assert ew.Layout.build(d, "k1", warp_size=4).dump() == g["k1"]
    assert ew.Layout.build(d, "k2", warp_size=4, threshold=1).dump() == g["k2"]
    g = golden["k2_100_8"]
    lay = ew.Layout.build(dev_csr(ew, _m(g["matrix"])), "k2", threshold=10).export()
    assert lay.reduction[0] == 16 and lay.rows_in_warp[0] == 1 and lay.maxrows[0] == 7
    assert (lay.reduction[1:] == 1).all()


@pytest.mark.parametrize("case", range(30))
def test_build_matches_oracle(ew, R, F, case):
    m = F.random_case(case)
    a = dev_csr(ew, m)
    fr, ir = R.sort_rows_desc(m)
    fd, idv = a.sort_rows_desc()
    assert np.array_equal(fr, fd) and np.array_equal(ir, idv)
    for ws in (4, 8, 32):
        got = ew.Layout.build(a, "k1", warp_size=ws)
        want = R.build_k1(m, warp_size=ws)
        assert_layout_equal(got.export(), want, K1_FIELDS)
        assert np.array_equal(got.value_slot_map(a), R.value_slot_map(want, m))
        R.free(want)
        for sort_rows in (True, False):
            got = ew.Layout.build(a, "k1", warp_size=ws, sort_rows=sort_rows)
            want = R.build_k1(m, warp_size=ws, sort_rows=sort_rows)
            assert_layout_equal(got.export(), want, K1_FIELDS)
            R.free(want)
        lens = np.diff(m.row_offsets)
        for t in sorted({1, 2, 3, max(1, int(lens.max()) // 3), max(1, int(lens.max()))}):
            got = ew.Layout.build(a, "k2", warp_size=ws, threshold=t)
            want = R.build_k2(m, t, warp_size=ws)
            assert_layout_equal(got.export(), want, K2_FIELDS)
            assert np.array_equal(got.value_slot_map(a), R.value_slot_map(want, m))
            R.free(want)
    if m.nrows == m.ncols:
        for rs in (False, True):
            got, fwd = a.reorder(rs)
            want, fwd_w = R.reorder(m, rs)
            ro, ci, v = got.export()
            assert np.array_equal(fwd, fwd_w)
            assert np.array_equal(ro, want.row_offsets)
            assert np.array_equal(ci, want.col_indices) and np.array_equal(v, want.values)


def test_unaligned_and_segment_sizes(ew, R, F):
    m = F.fem_tet_graph(1500, 5, 21, 2)
    a = dev_csr(ew, m)
    for seg, align in ((128, False), (64, True), (256, True)):
        got = ew.Layout.build(a, "k1", segment_bytes=seg, align=align).export()
        want = R.build_k1(m, segment_bytes=seg, align=align)
        assert_layout_equal(got, want, K1_FIELDS)
        got = ew.Layout.build(a, "k2", threshold=7, segment_bytes=seg, align=align).export()
        want = R.build_k2(m, 7, segment_bytes=seg, align=align)
        assert_layout_equal(got, want, K2_FIELDS)


def test_import_round_trip_and_refresh(ew, R, F):
    m = F.fem_tet_graph(900, 5, 21, 4)
    x = F.random_vector(m.ncols, 9)
    a = dev_csr(ew, m)
    for kind, t in (("k1", 0), ("k2", 6)):
        lay = ew.Layout.build(a, kind, threshold=t)
        e = lay.export()
        imp = ew.Layout.import_arrays(kind, 32, e.nrows, e.ncols, e.nnz, e.values, e.col_indices, e.warp_offset,
                                      e.maxrows, e.rows_in_warp, e.forward, e.sorted_row_length,
                                      reduction=e.reduction, rows_offset_warp=e.rows_offset_warp, threshold=t)
        assert np.array_equal(imp.spmv(x), lay.spmv(x))
        assert imp.dump() == lay.dump()
        # values-only refresh through the slot map (warp_layout.hpp:85-90)
        v2 = m.values * 2.0 + 1.0
        b = ew.Csr(m.nrows, m.ncols, m.row_offsets, m.col_indices, v2)
        lay.refresh_values(b)
        fresh = ew.Layout.build(b, kind, threshold=t)
        assert np.array_equal(lay.export().values, fresh.export().values)
    with pytest.raises(ValueError):
        ew.Layout.import_arrays("k1", 32, 3, 3, 1, [1.0], [0], [0], [5], [3], [0, 1, 1], [1, 0, 0])


@pytest.mark.parametrize("kid", ["csr_ref", "k1", "k2", "k1r", "k1rs", "k2r", "k2rs", "csr_vector", "coo"])
def test_kernel_values_refresh(ew, F, kid):
    """Values-only refresh of a prepared kernel (the paper's reorder once per
    Newton iteration): same structure, new values -> the
    refreshed kernel equals one prepared from scratch, bit for bit."""
    from tests.gpu_helpers import same

    m = F.fem_tet_graph(1200, 5, 21, 9)
    x = F.random_vector(m.ncols, 4)
    a = dev_csr(ew, m)
    k = ew.Kernel(kid, a, threshold=5)
    v2 = np.sin(np.arange(m.nnz)) + 2.0
    b = ew.Csr(m.nrows, m.ncols, m.row_offsets, m.col_indices, v2)
    k.refresh_values(b)
    fresh = ew.Kernel(kid, b, threshold=5)
    assert same(k.apply(x), fresh.apply(x)), kid
    if k.has_perm:
        assert same(k.apply_permuted(x), fresh.apply_permuted(x))
    # the prepared kernel owns its matrix: updating the source handle later
    # does not reach it (kernels.cpp:65-68 copies the matrix)
    b.update_values(v2 * 3.0)
    assert same(k.apply(x), fresh.apply(x))


def test_kernel_stored_slots(ew, R, F):
    """PreparedKernel::stored_slots (kernels.cpp:63, 104, 112) and padding claims
    (acceptance.cpp criterion 3): sorted K1 pads less than unsorted."""
    heart = F.fem_tet_graph(3129, 5, 21, 1)
    a = dev_csr(ew, heart)
    s = ew.Layout.build(a, "k1").export()
    u = ew.Layout.build(a, "k1", sort_rows=False).export()
    assert s.padded_slots < u.padded_slots
    assert ew.Kernel("k1", a).stored_slots == s.stored_slots
    assert ew.Kernel("csr_ref", a).stored_slots == heart.nnz

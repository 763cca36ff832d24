"""The reference-facing host API: the C++ drop-in (namespace ellwarp) and its
pybind11 module `_ellwarp` (proj/bindings/module.cpp names and defaults).

CPU: the module loads, and the seeded generators reproduce the reference's
matrices exactly (synth.cpp:10-214, compared with oracle/_ref).
GPU: the reference's own unit-test sources (proj/tests/test_ellwarp.cpp,
test_solver.cpp), compiled unchanged against our headers by
tests/cpp/Makefile, run against the device library; and the assertions of
proj/python/tests/test_smoke.py through `_ellwarp`."""
import math
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT_BIN = os.path.join(ROOT, "tests", "cpp", "_bin", "reference_unit_tests")


@pytest.fixture(scope="module")
def ew_mod():
    from paper_1501_00324_b200 import load_ellwarp

    return load_ellwarp()


def same_csr(a, b):
    return (a.nrows == b.nrows and a.ncols == b.ncols and list(a.row_offsets) == b.row_offsets.tolist()
            and list(a.col_indices) == b.col_indices.tolist()
            and np.array_equal(np.asarray(a.values, np.float64).view(np.int64), b.values.view(np.int64)))


def test_generators_match_reference(ew_mod, F):
    assert same_csr(ew_mod.laplacian3d(4, 5, 3), F.laplacian3d(4, 5, 3))
    assert same_csr(ew_mod.uniform_band(40, 7), F.uniform_band(40, 7))
    for n, lo, hi, seed in ((600, 5, 21, 12), (3129, 5, 21, 1), (200, 2, 9, 7), (50, 5, 50, 3)):
        assert same_csr(ew_mod.fem_tet_graph(n, lo, hi, seed), F.fem_tet_graph(n, lo, hi, seed)), (n, seed)
    for args in ((300, 1.5, 120, 3, 0), (500, 1.5, 100, 9, 0), (200, 1.2, 100, 11, 0), (64, 0.8, 64, 5, 40),
                 (1000, 2.0, 4700, 1, 0)):
        assert same_csr(ew_mod.powerlaw_rows(*args), F.powerlaw_rows(*args)), args
    for spec in ("laplacian3d:3,4,5", "fem_tet_graph:n=300,minrow=5,maxrow=21,seed=2",
                 "powerlaw_rows:nrows=200,alpha=1.5,maxrow=64,seed=4", "uniform_band:n=64,row_len=5"):
        assert same_csr(ew_mod.generate_synthetic(spec), F.generate(spec)), spec
    with pytest.raises(ValueError):
        ew_mod.generate_synthetic("bogus:1")
    with pytest.raises(ValueError):
        ew_mod.fem_tet_graph(10, 1, 5, 1)


def test_host_entry_points(ew_mod):
    assert ew_mod.kernel_ids() == ["csr_ref", "csr_vector", "coo", "ell", "hyb", "k1", "k1r", "k1rs", "k2",
                                   "k2r", "k2rs"]
    assert ew_mod.compute_k2_lanes(11, 10, 32) == 2
    assert ew_mod.compute_k2_lanes(400, 10, 32) == 32
    assert ew_mod.compute_alpha(10.0, 1.0, 2.0) == 10
    assert ew_mod.compute_alpha(0.0, 2.0, 2.0) is None
    s = ew_mod.matrix_stats(ew_mod.laplacian3d(3, 3, 3))
    assert s["nnz"] == 135 and s["bytes"] == 20 * 135 and s["minrow"] == 4 and s["maxrow"] == 7
    assert sum(s["histogram"].values()) == 27


@pytest.mark.gpu
def test_reference_cpp_unit_tests(ew):
    """proj/tests/test_ellwarp.cpp + test_solver.cpp, compiled unchanged."""
    if not os.path.exists(UNIT_BIN):
        pytest.skip("tests/cpp/_bin/reference_unit_tests not built (needs /root/reference)")
    out = subprocess.run([UNIT_BIN], capture_output=True, text=True, timeout=600)
    failed = [ln[7:] for ln in out.stdout.splitlines() if ln.startswith("[FAIL]")]
    print(out.stdout[-3000:], out.stderr[-3000:])
    assert "test cases:" in out.stdout
    assert failed == [], failed


# ---- proj/python/tests/test_smoke.py, through _ellwarp ------------------------


def close(a, b, tol=1e-12):
    return abs(a - b) <= tol * max(1.0, abs(a), abs(b))


@pytest.mark.gpu
def test_smoke_construct_and_stats(ew_mod, ew):
    m = ew_mod.SparseCsr.from_coo(3, 3, [0, 1, 2, 2], [0, 1, 0, 2], [2.0, 3.0, 1.0, 4.0])
    assert m.nnz() == 4
    stats = ew_mod.matrix_stats(m)
    assert stats["nnz"] == 4 and stats["bytes"] == 80 and stats["minrow"] == 1 and stats["maxrow"] == 2
    with pytest.raises(ValueError):
        ew_mod.SparseCsr(2, 2, [0, 2, 2], [1, 0], [1.0, 1.0])


@pytest.mark.gpu
def test_smoke_matrix_market_roundtrip(ew_mod, ew, tmp_path):
    # test_smoke.py:23-28: symmetric storage expands, bogus header raises
    text = "%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n2 1 5.0\n2 2 1.0\n"
    m = ew_mod.parse_matrix_market(text)
    assert m.nnz() == 3 and m.col_indices == [1, 0, 1] and m.values == [5.0, 5.0, 1.0]
    with pytest.raises(Exception):
        ew_mod.parse_matrix_market("%%bogus\n")
    with pytest.raises(Exception):
        ew_mod.parse_matrix_market("%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n")
    import gzip

    body = "%%MatrixMarket matrix coordinate pattern general\n% comment\n3 3 2\n1 3\n3 1\n"
    (tmp_path / "p.mtx").write_text(body)
    with gzip.open(tmp_path / "p.mtx.gz", "wt") as f:
        f.write(body)
    for name in ("p.mtx", "p.mtx.gz"):
        p = ew_mod.read_matrix_market(str(tmp_path / name))
        assert p.nrows == 3 and p.row_offsets == [0, 1, 1, 2] and p.col_indices == [2, 0] and p.values == [1.0, 1.0]


@pytest.mark.gpu
def test_smoke_device_kernels_match_reference(ew_mod, ew):
    m = ew_mod.fem_tet_graph(500, 5, 21, seed=7)
    x = [0.1 + 0.001 * i for i in range(m.ncols)]
    ref = ew_mod.spmv_reference(m, x)
    for kernel in ("csr_ref", "k1", "k1r", "k1rs", "k2", "k2r", "k2rs"):
        y = ew_mod.spmv(kernel, m, x, warp_size=32)
        assert all(close(a, b) for a, b in zip(y, ref)), kernel


@pytest.mark.gpu
def test_smoke_k2_threshold_sweep(ew_mod, ew):
    m = ew_mod.powerlaw_rows(200, 1.5, 64, seed=3)
    x = [1.0] * m.ncols
    ref = ew_mod.spmv_reference(m, x)
    maxrow = ew_mod.matrix_stats(m)["maxrow"]
    for t in (1, 4, maxrow):
        y = ew_mod.spmv("k2", m, x, threshold=t)
        assert all(close(a, b) for a, b in zip(y, ref))


@pytest.mark.gpu
def test_smoke_padding_ordering(ew_mod, ew):
    m = ew_mod.fem_tet_graph(1500, 5, 21, seed=2)
    ell = ew_mod.layout_info(m, "ell")
    k1 = ew_mod.layout_info(m, "k1")
    k1_unsorted = ew_mod.layout_info(m, "k1", sort_rows=False)
    assert k1["padded_slots"] <= ell["padded_slots"]
    assert k1["padded_slots"] < k1_unsorted["padded_slots"]


@pytest.mark.gpu
def test_smoke_reorder_worked_example(ew_mod, ew):
    offsets, cols, vals = [0], [], []
    lengths = [5, 7, 6, 5, 7, 5, 7]
    for r, ln in enumerate(lengths):
        if r == 0:
            cols += [0, 1, 3, 4, 5]
            vals += [7.0, 8.0, 9.0, 10.0, 2.0]
        else:
            cols += list(range(ln))
            vals += [float(10 * r + j) for j in range(ln)]
        offsets.append(len(cols))
    m = ew_mod.SparseCsr(7, 7, offsets, cols, vals)
    fwd, inv = ew_mod.sort_rows_desc(m)
    assert fwd == [1, 4, 6, 2, 0, 3, 5]
    reordered, fwd2 = ew_mod.reorder(m, sort_within_rows=True)
    assert fwd2 == fwd
    lo, hi = reordered.row_offsets[0], reordered.row_offsets[1]
    assert reordered.col_indices[lo:hi] == [0, 1, 4, 5, 6]
    assert reordered.values[lo:hi] == [8.0, 10.0, 7.0, 9.0, 2.0]
    r_only, _ = ew_mod.reorder(m)
    assert r_only.col_indices[:5] == [4, 0, 5, 1, 6]


@pytest.mark.gpu
def test_smoke_cg_and_alpha(ew_mod, ew):
    m = ew_mod.laplacian3d(5, 5, 5)
    b = ew_mod.spmv_reference(m, [1.0] * 125)
    res = ew_mod.cg_solve(m, b, kernel="k1rs", tol=1e-8)
    assert res["converged"]
    assert all(close(v, 1.0, 1e-6) for v in res["solution"])
    assert res["spmv_calls"] == res["iterations"] + 1 + res["iterations"] // 50
    assert ew_mod.compute_alpha(10.0, 1.0, 2.0) == 10


@pytest.mark.gpu
def test_resident_prepared_kernel(ew_mod, ew, R, F):
    import torch

    from oracle.oracle import Csr

    m = ew_mod.fem_tet_graph(2000, 5, 21, 3)
    k = ew_mod.prepare_kernel("k1rs", m)
    x = np.linspace(0.1, 1.0, m.ncols)
    y = k.apply(x)
    mo = Csr.make(m.nrows, m.ncols, m.row_offsets, m.col_indices, m.values)
    assert np.allclose(y, R.spmv_csr(mo, x), rtol=1e-12, atol=0)
    fwd, inv = k.perm
    yp = k.apply_permuted(x[fwd])
    assert np.array_equal(yp[inv], y)
    xd = torch.tensor(x, device="cuda")
    yd = torch.empty(m.nrows, dtype=torch.float64, device="cuda")
    k.apply_device(xd.data_ptr(), yd.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert np.array_equal(yd.cpu().numpy(), y)
    b = ew_mod.spmv_reference(m, [1.0] * m.ncols)
    d = ew_mod.extract_diagonal(m)
    res = k.cg_solve(np.asarray(b), d, permuted=True)
    ref = R.cg_csr(mo, b)
    assert res["iterations"] == ref.iterations
    h = np.asarray(res["residual_history"])
    assert np.all(np.abs(h - ref.residual_history) <= 1e-10 * (1 + ref.residual_history))
    assert math.isclose(res["solution"][0], 1.0, rel_tol=1e-6)


@pytest.mark.gpu
def test_prepare_kernel_locality_row_order(ew_mod, ew, R):
    """KernelOptions::row_order = locality through the C++ API / _ellwarp:
    same row sums as the reference kernel, CG within the comparator."""
    from oracle.oracle import Csr

    m = ew_mod.laplacian3d(9, 8, 7)
    mo = Csr.make(m.nrows, m.ncols, m.row_offsets, m.col_indices, m.values)
    x = np.linspace(0.1, 1.0, m.ncols)
    for kid in ("k1r", "k1rs"):
        k = ew_mod.prepare_kernel(kid, m, row_order="locality")
        assert np.array_equal(k.apply(x), ew_mod.prepare_kernel(kid, m).apply(x))
        b = ew_mod.spmv_reference(m, [1.0] * m.ncols)
        res = k.cg_solve(np.asarray(b), ew_mod.extract_diagonal(m), permuted=True)
        ref = R.cg_csr(mo, b)
        assert res["iterations"] == ref.iterations
        h = np.asarray(res["residual_history"])
        assert np.all(np.abs(h - ref.residual_history) <= 1e-10 * (1 + ref.residual_history))
    with pytest.raises(ValueError):
        ew_mod.prepare_kernel("k1", m, row_order="locality")

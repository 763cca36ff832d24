"""Parity at BASELINE.json's full sizes (configs 2 and 4 on one B200).

The C restatement (oracle/ew_oracle.c) runs the reference's layouts and K1
sums at these sizes in seconds, so the SpMV checks stay bitwise; the CG is
checked through size-independent properties (a 1000-iteration CPU solve of
config 4 takes minutes): true residual of the returned solution, agreement
of the last history entry with it, the exact-solution recovery for b = A 1,
and equality of the permuted / locality solves' iteration counts."""
import numpy as np
import pytest

from oracle.oracle import Csr
from tests.gpu_helpers import bits, rel_close

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def c2():
    from paper_1501_00324_b200 import workloads as W

    n, _, ro, ci, v = W.elasticity_box(86, 86, 86)
    return Csr.make(n, n, ro, ci, v)


@pytest.fixture(scope="module")
def c4():
    from paper_1501_00324_b200 import workloads as W

    n, _, ro, ci, v = W.ventricle_box(170, 170, 170)
    return Csr.make(n, n, ro, ci, v)


def dev(ew, m):
    return ew.Csr(m.nrows, m.ncols, m.row_offsets, m.col_indices, m.values)


def test_config2_k1_bitwise(ew, R, c2):
    """The default bench's kernel (16-bit columns at this size) against the
    restated reference K1, bit for bit, through host and device buffers;
    linearity and the layout's padding count as size-independent checks."""
    a = dev(ew, c2)
    x = np.random.default_rng(1).uniform(0.1, 1.0, c2.ncols)
    k = ew.Kernel("k1", a)
    y = k.apply(x)
    lay = R.build_k1(c2)
    try:
        want = R.spmv_layout(lay, x, scatter=True)
        assert k.stored_slots == lay.stored_slots
    finally:
        R.free(lay)
    assert np.array_equal(bits(y), bits(want))
    assert rel_close(y, R.spmv_csr(c2, x), 1e-12)
    # host buffers run the row-block pipeline; device buffers the whole
    # layout, with 16-bit columns on every warp of this matrix
    import torch

    assert k.info().narrow_slots >= 0.99 * k.stored_slots
    yd = k.apply(torch.tensor(x, device="cuda")).cpu().numpy()
    assert np.array_equal(bits(yd), bits(want))
    x2 = np.random.default_rng(2).uniform(-1.0, 1.0, c2.ncols)
    lhs = k.apply(2.0 * x + x2)
    rhs = 2.0 * y + k.apply(x2)
    assert np.allclose(lhs, rhs, rtol=1e-12, atol=1e-12 * np.abs(rhs).max())


def test_config4_k1rs_both_row_orders(ew, R, c4):
    """k1rs on the randomly renumbered ventricle mesh: the reference row
    order bitwise against the restated reference; the locality order row for
    row equal to it (same entry order per row)."""
    a = dev(ew, c4)
    x = np.random.default_rng(3).uniform(0.1, 1.0, c4.ncols)
    y_ref_order = ew.Kernel("k1rs", a).apply(x)
    op, _ = R.reorder(c4, True)
    lay = R.build_k1(op)
    try:
        want = R.spmv_layout(lay, x[lay.forward], scatter=True)
    finally:
        R.free(lay)
    assert np.array_equal(bits(y_ref_order), bits(want))
    k = ew.Kernel("k1rs", a, row_order="locality")
    assert np.array_equal(k.apply(x), want)
    fwd, inv = k.perm()
    assert np.array_equal(np.sort(fwd), np.arange(c4.nrows))
    assert np.array_equal(k.apply_permuted(x[fwd])[inv], want)


def test_config4_cg_properties(ew, R, c4):
    """Jacobi PCG on config 4 to tol 1e-8 (b = A 1): converged, the true
    residual of the returned solution is at the tolerance, and the reference
    and locality row orders reach 1e-6 within 1% of the same iteration. (The
    total, ~2,450 iterations, varies by a few percent: the dot products round
    differently and the last hundreds of iterations creep along a plateau
    near 1e-8, where the stopping iteration is rounding-sensitive.)"""
    a = dev(ew, c4)
    diag = a.extract_diagonal()
    b = a.spmv(np.ones(c4.ncols))
    runs = {}
    for order in ("reference", "locality"):
        k = ew.Kernel("k1rs", a, row_order=order)
        res = k.cg_solve(b, diag, permuted=True, max_iterations=5000)
        assert res.converged, order
        assert res.spmv_calls == 1 + res.iterations + res.iterations // 50
        r = b - a.spmv(res.solution)
        true_rel = np.linalg.norm(r) / np.linalg.norm(b)
        assert true_rel <= 1e-7, (order, true_rel)
        assert res.residual_history[-1] <= 1e-8
        assert np.all(np.isfinite(res.residual_history))
        runs[order] = res
    first = {o: int(np.argmax(r.residual_history <= 1e-6)) for o, r in runs.items()}
    assert abs(first["reference"] - first["locality"]) <= max(1, first["reference"] // 100), first
    its = runs["reference"].iterations
    assert abs(its - runs["locality"].iterations) <= max(1, its // 20)
    assert np.allclose(runs["reference"].solution, runs["locality"].solution, rtol=1e-6, atol=1e-6)


@pytest.mark.parametrize("transport", ["copy", "peer"])
def test_config2_partitioned_spmv_bitwise(ew, c2, transport):
    """Config 2 in 4 row blocks on one GPU (interior rows overlapping the
    halo, boundary rows after it): bitwise the single-GPU K1."""
    a = dev(ew, c2)
    x = np.random.default_rng(4).uniform(0.1, 1.0, c2.ncols)
    single = ew.Kernel("k1", a).apply(x)
    d = ew.Dist.local(c2, 4, transport=transport)
    y = d.spmv(x)
    both_zero = (y == 0) & (single == 0)
    assert np.all(both_zero | (bits(y) == bits(single)))


def _first_cross(h, ref, thr):
    n = min(len(h), len(ref))
    d = np.abs(h[:n] - ref[:n]) / (1.0 + ref[:n])
    i = np.flatnonzero(d > thr)
    return int(i[0]) if i.size else n


@pytest.mark.parametrize("transport", ["peer", "copy"])
def test_config5_scaled_partitioned_cg_vs_oracle(ew, R, transport):
    """The partitioned PCG (4 row blocks, the multi-GPU code path with the
    in-process peer transport or device copies) on config 5's operator at a
    test size (3-DOF elasticity box(40,40,40), 206,763 rows), 400 forced
    iterations, against the restated reference: cg_solve over the K1 layout
    of the whole matrix (threaded restatement, bitwise the reference). The
    partitions' dot products are summed in rank order (a different order
    than the reference's sequential sums), so the history is held to the
    bar the reference meets against itself with a different summation
    order: its own cg_solve_permuted over k1rs vs cg_solve over K1
    (test_solver.cpp:83-112), which itself leaves the comparator
    |dh| <= 1e-10 (1 + h) at iteration ~219 (CG amplifies rounding
    differences: the device K1 solve, the 2- and 4-way partitions and the
    device k1rs solve all leave it at 193-201). Held: the comparator over
    the first 3/4 of the pair's in-comparator span, every deviation
    threshold reached no earlier than 3/4 of where the pair reaches it,
    1 + it + it/50 SpMVs, solution within 1e-9."""
    import os

    from paper_1501_00324_b200 import workloads as W

    n, _, ro, ci, v = W.elasticity_box(40, 40, 40)
    m = Csr.make(n, n, ro, ci, v)
    b = R.spmv_csr(m, np.ones(n))
    diag = R.extract_diagonal(m)
    lay = R.build_k1(m)
    th = os.cpu_count() or 1
    try:
        ref = R.cg_layout(lay, b, diag=diag, tol=1e-300, max_iterations=400, threads=th)
    finally:
        R.free(lay)
    op, _ = R.reorder(m, True)
    lay = R.build_k1(op)
    try:
        perm = R.cg_layout(lay, b, diag=diag, permuted=True, tol=1e-300, max_iterations=400, threads=th)
    finally:
        R.free(lay)
    d = ew.Dist.local(m, 4, transport=transport)
    res = d.cg_solve(b, diag, tol=1e-300, max_iterations=400)
    assert res.iterations == 400 and res.spmv_calls == 1 + 400 + 8
    h, hk, hp = res.residual_history, ref.residual_history, perm.residual_history
    dev = np.abs(h - hk) / (1.0 + hk)
    own_dev = np.abs(hp - hk) / (1.0 + hk)
    msg = f"max deviation {dev.max():.2e} (reference's own k1rs-vs-K1: {own_dev.max():.2e})"
    own = int(0.75 * _first_cross(hp, hk, 1e-10))
    assert np.all(dev[:own] <= 1e-10), msg
    for thr in (1e-10, 1e-8, 1e-6):
        assert _first_cross(h, hk, thr) >= 0.75 * _first_cross(hp, hk, thr), (thr, msg)
    assert np.max(np.abs(res.solution - ref.solution)) <= 1e-9 * max(1.0, np.abs(ref.solution).max())

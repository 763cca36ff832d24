"""Locality row order for the r / rs kernels (ew_kernel_options.row_order =
EW_ROW_ORDER_LOCALITY, csrc/ew_order.cu).

The order is an extension (the reference has only sort_rows_desc,
permutation.cpp:49-55), so its contract is checked three ways:
  * the permutation equals a plain-Python restatement of the device rule
    (Cuthill-McKee BFS, then the reference's stable longest-first sort);
  * K1: every row sum equals the reference kernel's (each row keeps the
    reference's entry order: original for r, ascending sorted index for rs,
    reorder.cpp:8-43) -- compared with ==, since a row may carry a different
    number of +0.0 padding terms than in the reference's warp;
  * K2: a row's lane chunks are `maxrows` of its warp long
    (warp_spmv.cpp:73-99), so the chunking -- and the rounding -- follows its
    warp-mates; rows are checked with the reference's kernel tolerance,
    1e-12 relative per entry (acceptance.cpp:144-186);
  * CG in the locality numbering meets the reference comparator
    |h - h_ref| <= 1e-10 (1 + h_ref) over the same iteration count
    (test_solver.cpp:109-110).
"""
import numpy as np
import pytest

from oracle.oracle import Csr
from paper_1501_00324_b200 import workloads as W
from tests.gpu_helpers import oracle_apply, rel_close

pytestmark = pytest.mark.gpu

MAX_RESTARTS = 64


def locality_order(ro, ci, n):
    """Restatement of ew::locality_order (ew_order.cu)."""
    seen = np.zeros(n, bool)
    order = []
    lens = np.diff(ro)
    restarts = 0
    while len(order) < n and restarts < MAX_RESTARTS:
        cand = np.flatnonzero(~seen)
        start = int(cand[np.lexsort((cand, lens[cand]))[0]])  # (degree, id)
        order.append(start)
        seen[start] = True
        restarts += 1
        head = len(order) - 1
        while head < len(order):
            tail = len(order)
            parent = {}
            for pos in range(head, tail):
                r = order[pos]
                for u in ci[ro[r]:ro[r + 1]]:
                    u = int(u)
                    if u < n and not seen[u] and u not in parent:
                        parent[u] = pos  # frontier scanned in position order: first = min
            head = tail
            for u in sorted(parent, key=lambda u: (parent[u], u)):
                order.append(u)
                seen[u] = True
            if not parent:
                break
    order.extend(int(r) for r in np.flatnonzero(~seen))
    order = np.asarray(order, np.int64)
    # stable longest-first sort of the BFS order
    return order[np.argsort(-lens[order], kind="stable")]


def dev(ew, m):
    return ew.Csr(m.nrows, m.ncols, m.row_offsets, m.col_indices, m.values)


def cases(F):
    n, _, ro, ci, v = W.ventricle_box(7, 6, 5)
    yield "ventricle", Csr.make(n, n, ro, ci, v)
    yield "laplacian", F.laplacian3d(6, 5, 4)
    yield "powerlaw", F.powerlaw_rows(400, 1.5, 60, 5, 400)
    yield "band", F.uniform_band(300, 5)
    for i in range(6):
        m = F.random_case(i)
        if m.nrows == m.ncols:
            yield f"random{i}", m


def _block_diagonal(nblocks, size, seed):
    """nblocks disconnected path graphs (SPD tridiagonal blocks), shuffled."""
    n = nblocks * size
    rows, cols = [], []
    for b in range(nblocks):
        for i in range(size):
            r = b * size + i
            for c in (r - 1, r, r + 1):
                if b * size <= c < (b + 1) * size:
                    rows.append(r)
                    cols.append(c)
    perm = np.random.default_rng(seed).permutation(n)
    rows, cols = perm[np.array(rows)], perm[np.array(cols)]
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    ro = np.zeros(n + 1, np.int64)
    np.add.at(ro, rows + 1, 1)
    ro = np.cumsum(ro)
    vals = np.where(rows == cols, 4.0, -1.0)
    return Csr.make(n, n, ro, cols.astype(np.int64), vals)


def test_edge_cases(ew, R, F):
    """Empty rows, one row, and more components than the BFS restarts
    (the rest is appended in row order)."""
    cases_ = [("components", _block_diagonal(100, 3, 1)), ("one", Csr.make(1, 1, [0, 1], [0], [2.0]))]
    m = F.random_csr(60, 60, 0.05, 8, empty=0.3)
    cases_.append(("empty_rows", m))
    for name, m in cases_:
        a = dev(ew, m)
        x = F.random_vector(m.ncols, 3)
        for kid in ("k1r", "k1rs"):
            k = ew.Kernel(kid, a, row_order="locality")
            fwd, _ = k.perm()
            assert np.array_equal(fwd, locality_order(m.row_offsets, m.col_indices, m.nrows)), (name, kid)
            assert np.array_equal(k.apply(x), oracle_apply(R, kid, m, x)), (name, kid)


def test_order_matches_restatement(ew, F):
    for name, m in cases(F):
        a = dev(ew, m)
        for kid in ("k1r", "k1rs", "k2r", "k2rs"):
            k = ew.Kernel(kid, a, threshold=3, row_order="locality")
            fwd, inv = k.perm()
            want = locality_order(m.row_offsets, m.col_indices, m.nrows)
            assert np.array_equal(fwd, want), (name, kid)
            assert np.array_equal(inv[fwd], np.arange(m.nrows)), (name, kid)


def test_row_sums_equal_reference(ew, R, F):
    for name, m in cases(F):
        x = F.random_vector(m.ncols, 11)
        a = dev(ew, m)
        for kid in ("k1r", "k1rs", "k2r", "k2rs"):
            for t in (2, 5, 0):
                k = ew.Kernel(kid, a, threshold=t, row_order="locality")
                want = oracle_apply(R, kid, m, x, 32, t)
                y = k.apply(x)
                fwd, _ = k.perm()
                yp = k.apply_permuted(x[fwd])
                if kid.startswith("k1"):
                    assert np.array_equal(y, want), (name, kid, t)
                    assert np.array_equal(yp, want[fwd]), (name, kid, t)
                else:
                    assert rel_close(y, want, 1e-12), (name, kid, t)
                    assert rel_close(yp, want[fwd], 1e-12), (name, kid, t)
                    assert rel_close(y, R.spmv_csr(m, x), 1e-12), (name, kid, t)


def test_refresh_values(ew, R, F):
    n, _, ro, ci, v = W.ventricle_box(6, 6, 6)
    m = Csr.make(n, n, ro, ci, v)
    a = dev(ew, m)
    x = F.random_vector(n, 5)
    m2 = Csr.make(n, n, ro, ci, v * 1.5 + 0.25)
    a2 = dev(ew, m2)
    for kid in ("k1r", "k1rs", "k2rs"):
        k = ew.Kernel(kid, a, threshold=4, row_order="locality")
        k.refresh_values(a2)
        y, want = k.apply(x), oracle_apply(R, kid, m2, x, 32, 4)
        assert np.array_equal(y, want) if kid.startswith("k1") else rel_close(y, want, 1e-12), kid


def test_cg_histories(ew, R, F):
    """Well-conditioned operators only: on the jittered ventricle stand-in the
    CG recurrence amplifies any rounding difference (even the reference's own
    k1r vs csr_ref histories part after ~100 iterations), so the comparator
    is applied where the reference applies it -- P1 Laplacians, here with a
    random renumbering so the locality order differs from every natural one."""
    n, _, ro, ci, v = W.laplacian_box(10, 9, 8)
    n, _, ro, ci, v = W.renumber(n, ro, ci, v, np.random.default_rng(3).permutation(n))
    for m in (Csr.make(n, n, ro, ci, v), F.laplacian3d(8, 8, 8)):
        b = R.spmv_csr(m, np.ones(m.nrows))
        ref = R.cg_csr(m, b)
        a = dev(ew, m)
        diag = a.extract_diagonal()
        for kid in ("k1r", "k1rs", "k2rs"):
            k = ew.Kernel(kid, a, threshold=4, row_order="locality")
            for permuted in (False, True):
                res = k.cg_solve(b, diag, permuted=permuted)
                assert res.converged and res.iterations == ref.iterations, (kid, permuted)
                assert res.spmv_calls == ref.spmv_calls
                h, hr = res.residual_history, ref.residual_history
                assert np.all(np.abs(h - hr) <= 1e-10 * (1 + hr)), (kid, permuted)
                assert np.allclose(res.solution, ref.solution, rtol=1e-10, atol=1e-12)


def test_locality_needs_reordered_id(ew, F):
    a = dev(ew, F.laplacian3d(3, 3, 3))
    for kid in ("k1", "k2", "csr_ref", "ell"):
        with pytest.raises(ValueError):
            ew.Kernel(kid, a, row_order="locality")
    m = F.random_csr(5, 7, 0.5, 3)
    with pytest.raises(ValueError):
        ew.Kernel("k1r", dev(ew, m), row_order="locality")  # non-square

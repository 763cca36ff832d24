"""CG parity at BASELINE.json's config 4 (5,000,211 rows, 74.3M nonzeros,
Jacobi PCG, b = A 1) against the REAL reference's residual histories.

The fixtures tests/golden/c4_cg_{k1rs,csr_ref}.npz hold the histories of the
reference's own cg_solve_permuted over prepare_kernel("k1rs") and cg_solve
over csr_ref (oracle/_ref, the reference compiled from its sources; made by
tests/golden/make_c4_cg.py, ~1 h each on one core), tol 1e-8.

What parity can mean here is set by the reference itself: its k1rs and
csr_ref solves differ only in summation order (row sums of the reordered
rows, dot products over permuted vectors), yet their histories leave the
reference's own comparator |dh| <= 1e-10 (1 + h) (test_solver.cpp:104-112) at
iteration 244, pass 1e-6 at 406, differ by O(1) in mid-solve, and stop at
2,430 vs 2,449 iterations. CG on this jittered, randomly numbered mesh
amplifies a rounding difference ~10x every ~40 iterations. So the device
solve is held to the bar the reference meets against itself:

  * the first 200 history entries within the reference comparator;
  * every deviation threshold (1e-10, 1e-8, 1e-6) first crossed no earlier
    than 3/4 of the iteration where the reference's own pair crosses it;
  * a forced 1000-iteration solve does exactly 1000 iterations and 1021
    SpMVs (1 + it + it/50, test_solver.cpp:55);
  * the tol-1e-8 solve converges within the reference pair's iteration
    spread (|it - it_k1rs| <= 2 |it_k1rs - it_csr| + 10), and its solution
    equals the reference's within 1e-9 at 257 sampled rows (the reference's
    own pair: 5.7e-11)."""
import hashlib
import os

import numpy as np
import pytest

from oracle.oracle import Csr

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.fixture(scope="module")
def fixtures():
    return {k: np.load(os.path.join(GOLDEN, f"c4_cg_{k}.npz")) for k in ("k1rs", "csr_ref")}


@pytest.fixture(scope="module")
def c4(R, fixtures):
    from paper_1501_00324_b200 import workloads as W

    n, _, ro, ci, v = W.ventricle_box(170, 170, 170)
    m = Csr.make(n, n, ro, ci, v)
    assert digest(m.row_offsets, m.col_indices, m.values) == str(fixtures["k1rs"]["matrix_sha256"]), \
        "config 4 generated differently here than where the fixture was made"
    b = R.spmv_csr(m, np.ones(n))  # b = A 1 (tools/ellwarp_cli.cpp:192-195)
    assert digest(b) == str(fixtures["k1rs"]["b_sha256"])
    return m, b


def first_cross(h, ref, thr):
    n = min(len(h), len(ref))
    d = np.abs(h[:n] - ref[:n]) / (1.0 + ref[:n])
    i = np.flatnonzero(d > thr)
    return int(i[0]) if i.size else n


@pytest.fixture(scope="module")
def kernels(ew, c4):
    m, _ = c4
    a = ew.Csr(m.nrows, m.ncols, m.row_offsets, m.col_indices, m.values)
    return a, {o: ew.Kernel("k1rs", a, row_order=o) for o in ("reference", "locality")}


@pytest.mark.parametrize("order", ["reference", "locality"])
def test_config4_forced_1000_iterations(c4, fixtures, kernels, order):
    m, b = c4
    a, ks = kernels
    res = ks[order].cg_solve(b, a.extract_diagonal(), permuted=True, tol=1e-300, max_iterations=1000)
    assert res.iterations == 1000 and not res.converged
    assert res.spmv_calls == 1021
    h = res.residual_history
    assert h.size == 1001 and np.all(np.isfinite(h))
    hk, hc = fixtures["k1rs"]["history"], fixtures["csr_ref"]["history"]
    # the first 200 entries: the reference comparator
    assert np.all(np.abs(h[:201] - hk[:201]) <= 1e-10 * (1.0 + hk[:201]))
    for thr in (1e-10, 1e-8, 1e-6):
        own = first_cross(hk, hc, thr)
        ours = first_cross(h, hk, thr)
        assert ours >= 0.75 * own, (thr, ours, own)


@pytest.mark.parametrize("order", ["reference", "locality"])
def test_config4_tol_1e8(c4, fixtures, kernels, order):
    m, b = c4
    a, ks = kernels
    res = ks[order].cg_solve(b, a.extract_diagonal(), permuted=True, tol=1e-8, max_iterations=5000)
    fk, fc = fixtures["k1rs"], fixtures["csr_ref"]
    it_k, it_c = int(fk["iterations"]), int(fc["iterations"])
    assert res.converged and res.residual_history[-1] <= 1e-8
    assert res.spmv_calls == 1 + res.iterations + res.iterations // 50
    assert abs(res.iterations - it_k) <= 2 * abs(it_k - it_c) + 10, (res.iterations, it_k, it_c)
    idx = fk["solution_idx"]
    assert np.max(np.abs(res.solution[idx] - fk["solution_samples"])) <= 1e-9
    assert np.max(np.abs(res.solution[idx] - fc["solution_samples"])) <= 1e-9
    assert abs(np.linalg.norm(res.solution) - float(fk["solution_norm"])) <= 1e-9 * float(fk["solution_norm"])

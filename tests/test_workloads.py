"""Config 3 (BASELINE.json configs[2]): the paper's 15-matrix suite at its
Table 2 sizes. Every stand-in must reproduce Table 2's
nz, nrows, minrow and maxrow (within 5%; all but Epidemiology's nz exactly)
and be a canonical CSR (strictly increasing columns per row). CPU only."""
import numpy as np
import pytest

from paper_1501_00324_b200 import workloads as W


@pytest.mark.parametrize("entry", W.TABLE2, ids=[t[0] for t in W.TABLE2])
def test_table2_standin_stats(entry):
    name, nnz, nrows, minrow, maxrow = entry
    n, nc, ro, ci, v = W.table2_matrix(name)
    lens = np.diff(ro)
    assert n == nrows and nc == nrows
    assert abs(int(ro[-1]) - nnz) <= 0.05 * nnz
    assert int(lens.min()) == minrow and int(lens.max()) == maxrow
    if name != "epidemiology":  # a 675 x 779 grid: 2,100,392 vs 2,100,225
        assert int(ro[-1]) == nnz
    rows = np.repeat(np.arange(n), lens)
    same_row = np.diff(rows) == 0
    assert np.all(np.diff(ci)[same_row] > 0)
    assert ci.min() >= 0 and ci.max() < nc and np.all(np.isfinite(v))


def test_table2_deterministic():
    a = W.table2_matrix("heart30k")
    b = W.table2_matrix("heart30k")
    assert all(np.array_equal(x, y) for x, y in zip(a[2:], b[2:]))

"""Generate tests/golden/golden.json from the REAL reference (oracle/_ref,
compiled from /root/reference/proj/src by oracle/Makefile).

Every literal the reference's own tests assert is re-checked here against the
compiled reference before it is written, so the fixture is pinned twice: by
the reference's test sources (file:line below) and by running the reference.

Run (in the container that has /root/reference):
    make -C oracle && python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Csr, Reference  # noqa: E402

F = Reference()


def csr_json(m):
    return dict(nrows=m.nrows, ncols=m.ncols, row_offsets=m.row_offsets.tolist(),
                col_indices=m.col_indices.tolist(), values=m.values.tolist())


def worked_example():
    # test_ellwarp.cpp:17-36 / acceptance.cpp:89-107 / test_smoke.py:75-94
    lengths = [5, 7, 6, 5, 7, 5, 7]
    ro, ci, v = [0], [], []
    for r, ln in enumerate(lengths):
        if r == 0:
            ci += [0, 1, 3, 4, 5]
            v += [7.0, 8.0, 9.0, 10.0, 2.0]
        else:
            ci += list(range(ln))
            v += [float(10 * r + j) for j in range(ln)]
        ro.append(len(ci))
    return Csr.make(7, 7, ro, ci, v)


def main():
    g = {}
    m = worked_example()
    fwd, inv = F.sort_rows_desc(m)
    assert fwd.tolist() == [1, 4, 6, 2, 0, 3, 5]  # test_ellwarp.cpp:55
    x = np.arange(1, 8, dtype=np.float64)
    r_op, _ = F.reorder(m, False)
    rs_op, _ = F.reorder(m, True)
    assert r_op.col_indices[:5].tolist() == [4, 0, 5, 1, 6]  # test_ellwarp.cpp:87
    assert rs_op.col_indices[:5].tolist() == [0, 1, 4, 5, 6]  # :101
    assert rs_op.values[:5].tolist() == [8.0, 10.0, 7.0, 9.0, 2.0]  # :102
    y = F.spmv_csr(m, x)
    assert y[0] == 121.0  # test_ellwarp.cpp:288
    g["worked"] = dict(matrix=csr_json(m), forward=fwd.tolist(), inverse=inv.tolist(),
                       x=x.tolist(), x_prime=x[fwd].tolist(), c_prime=r_op.col_indices[:5].tolist(),
                       c_second=rs_op.col_indices[:5].tolist(), a_second=rs_op.values[:5].tolist(),
                       y=y.tolist())
    assert g["worked"]["x_prime"] == [2, 5, 7, 3, 1, 4, 6]

    # test_ellwarp.cpp:40-48: lengths [1,3,2] -> forward [1,2,0]
    m = Csr.make(3, 3, [0, 1, 4, 6], [0, 0, 1, 2, 0, 1], [1.0] * 6)
    assert F.sort_rows_desc(m)[0].tolist() == [1, 2, 0]
    g["sort_132"] = dict(matrix=csr_json(m), forward=[1, 2, 0])

    # test_ellwarp.cpp:130-144: four rows, ws 4
    m = Csr.make(4, 4, [0, 4, 7, 9, 10], [0, 1, 2, 3, 0, 1, 2, 0, 1, 0], [1.0] * 10)
    lay = F.build("k1", m, warp_size=4)
    assert lay.nwarps == 1 and lay.maxrows.tolist() == [4] and lay.stored_slots == 16
    assert lay.padded_slots == 6
    g["k1_four_rows"] = dict(matrix=csr_json(m), warp_size=4, maxrows=[4], stored_slots=16,
                             padded_slots=6)

    # test_ellwarp.cpp:413-433: dump_layout golden text (pins the 32-slot alignment unit)
    m = Csr.make(6, 6, [0, 1, 4, 6, 7, 8, 9], [0, 0, 1, 2, 0, 1, 0, 0, 0], [1.0] * 9)
    k1_dump = ("k1 warp_size=4 nrows=6 nnz=9 nwarps=2\n"
               "warp 0: offset=0 maxrows=3 reduction=1 rows=[0,4)\n"
               "warp 1: offset=32 maxrows=1 reduction=1 rows=[4,6)\n")
    k2_dump = ("k2 warp_size=4 nrows=6 nnz=9 threshold=1 nwarps=3\n"
               "warp 0: offset=0 maxrows=1 reduction=4 rows=[0,1)\n"
               "warp 1: offset=32 maxrows=1 reduction=2 rows=[1,2)\n"
               "warp 2: offset=64 maxrows=1 reduction=1 rows=[2,6)\n")
    assert F.build("k1", m, warp_size=4).dump == k1_dump
    assert F.build("k2", m, warp_size=4, threshold=1).dump == k2_dump
    g["dump"] = dict(matrix=csr_json(m), k1=k1_dump, k2=k2_dump)

    # test_ellwarp.cpp:188-207 compute_k2_lanes
    lanes = []
    for nnz, t, ws, want in [(10, 10, 32, 1), (11, 10, 32, 2), (41, 10, 32, 8), (400, 10, 32, 32),
                             (0, 10, 32, 1)]:
        assert F.compute_k2_lanes(nnz, t, ws) == want
        lanes.append([nnz, t, ws, want])
    for nnz in (1, 5, 9, 17, 33, 64, 100, 319, 320, 321):
        for t in (1, 3, 10, 16):
            for ws in (4, 8, 32):
                lanes.append([nnz, t, ws, F.compute_k2_lanes(nnz, t, ws)])
    g["k2_lanes"] = lanes

    # test_ellwarp.cpp:221-239: rows [100, 8, 8, ...], T = 10
    ro, ci = [0], []
    for r in range(100):
        ln = 100 if r == 0 else 8
        ci += list(range(ln))
        ro.append(len(ci))
    m = Csr.make(100, 100, ro, ci, [1.0] * len(ci))
    lay = F.build("k2", m, threshold=10)
    assert lay.reduction[0] == 16 and lay.rows_in_warp[0] == 1 and lay.maxrows[0] == 7
    g["k2_100_8"] = dict(matrix=csr_json(m), threshold=10, reduction0=16, rows_in_warp0=1, maxrows0=7)

    # test_ellwarp.cpp:348-360: four lanes reduce to 255
    m = Csr.make(8, 8, [0, 8, 8, 8, 8, 8, 8, 8, 8], list(range(8)), [1, 2, 4, 8, 16, 32, 64, 128])
    lay = F.build("k2", m, threshold=2)
    assert lay.reduction[0] == 4
    y = F.apply("k2", m, np.ones(8), threshold=2)
    assert y[0] == 255.0
    g["four_lane"] = dict(matrix=csr_json(m), threshold=2, y0=255.0)

    # CG: test_solver.cpp:43-56 (laplacian 4^3, b = A*1) with the reference history
    cg = []
    for name, mat, b, kernel, permuted in [
        ("laplacian444", F.laplacian3d(4, 4, 4), None, "csr_ref", False),
        ("laplacian543", F.laplacian3d(5, 4, 3), None, "csr_ref", False),
        ("laplacian888_k1rs_perm", F.laplacian3d(8, 8, 8), None, "k1rs", True),
        ("femtet600", F.fem_tet_graph(600, 5, 21, 12), F.random_vector(600, 31), "csr_ref", False),
        ("femtet600_k1rs_perm", F.fem_tet_graph(600, 5, 21, 12), F.random_vector(600, 31), "k1rs", True),
    ]:
        if b is None:
            b = F.spmv_csr(mat, np.ones(mat.ncols))
        res = F.cg(kernel, mat, b, permuted=permuted)
        assert res.converged
        assert res.spmv_calls == res.iterations + 1 + res.iterations // 50
        cg.append(dict(name=name, kernel=kernel, permuted=permuted, matrix=csr_json(mat), b=b.tolist(),
                       iterations=res.iterations, spmv_calls=res.spmv_calls,
                       history=res.residual_history.tolist(), solution=res.solution.tolist()))
    g["cg"] = cg

    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(out, "w") as f:
        json.dump(g, f)
    print("wrote", out, os.path.getsize(out), "bytes")


if __name__ == "__main__":
    main()

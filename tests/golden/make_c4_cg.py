"""Generate the config-4 CG parity fixture (tests/golden/c4_cg_<kernel>.npz)
by running the REAL reference (oracle/_ref, compiled from
/root/reference/proj/src by oracle/Makefile) on BASELINE.json's config 4.

Config 4 = workloads.ventricle_box(170, 170, 170): 5,000,211 rows, 74.3M
nonzeros, b = A * 1 (tools/ellwarp_cli.cpp:192-195), Jacobi, tol 1e-8
(CgConfig defaults, cg.hpp:12-20), run to convergence (max 5000 iterations):
the first 1001 history entries are also the reference's history of a forced
1000-iteration solve (tol only decides when to stop, cg.cpp:92).

  k1rs     cg_solve_permuted over prepare_kernel("k1rs").apply_permuted
           (the benchmarked kernel; the reference's own row order)
  csr_ref  cg_solve over spmv_csr_reference (the unpermuted solve the
           reference's permuted-vs-plain comparator measures against,
           test_solver.cpp:104-112)

The fixture records sha256 digests of the matrix and b, so a test that
regenerates the matrix on another machine first proves it has the same
input. --impl restatement runs the C restatement (oracle/ew_oracle.c,
threaded SpMV, sequential dots) instead and checks it against an existing
fixture bit for bit, which pins the restatement at full size.

Run in the container that has /root/reference (single-threaded reference:
~20 minutes per kernel):
    make -C oracle && python tests/golden/make_c4_cg.py --kernel k1rs
"""
import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

HERE = os.path.dirname(os.path.abspath(__file__))
DIMS = (170, 170, 170)
TOL = 1e-8
MAX_IT = 5000


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def config4():
    from oracle.oracle import Csr
    from paper_1501_00324_b200 import workloads as W

    n, _, ro, ci, v = W.ventricle_box(*DIMS)
    return Csr.make(n, n, ro, ci, v)


def fixture_path(kernel):
    return os.path.join(HERE, f"c4_cg_{kernel}.npz")


def solution_samples(x):
    idx = np.linspace(0, x.size - 1, 257).astype(np.int64)
    return idx, x[idx]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernel", choices=["k1rs", "csr_ref"], default="k1rs")
    ap.add_argument("--impl", choices=["reference", "restatement"], default="reference")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    from oracle.oracle import Reference, Restatement

    t = time.time()
    m = config4()
    R = Restatement()
    b = R.spmv_csr(m, np.ones(m.ncols))
    print(f"config 4: {m.nrows} rows, {m.nnz} nnz ({time.time() - t:.0f}s)", flush=True)
    t = time.time()
    permuted = args.kernel == "k1rs"
    if args.impl == "reference":
        res = Reference().cg(args.kernel, m, b, tol=TOL, max_iterations=MAX_IT, permuted=permuted)
    else:
        diag = R.extract_diagonal(m)
        if permuted:
            op, _ = R.reorder(m, True)
            lay = R.build_k1(op)
            res = R.cg_layout(lay, b, diag=diag, permuted=True, tol=TOL, max_iterations=MAX_IT,
                              threads=args.threads)
            R.free(lay)
        else:
            res = R.cg_csr(m, b, tol=TOL, max_iterations=MAX_IT)
    dt = time.time() - t
    print(f"{args.impl} {args.kernel}: {res.iterations} iterations, converged {res.converged}, "
          f"{res.spmv_calls} SpMVs, {dt:.0f}s", flush=True)
    idx, xs = solution_samples(res.solution)
    if args.impl == "restatement":
        f = np.load(fixture_path(args.kernel))
        same = (np.array_equal(f["history"].view(np.int64), res.residual_history.view(np.int64))
                and str(f["solution_sha256"]) == digest(res.solution))
        print("restatement == reference fixture bit for bit:", same, flush=True)
        sys.exit(0 if same else 1)
    meta = {"dims": DIMS, "nrows": m.nrows, "nnz": m.nnz, "tol": TOL, "max_iterations": MAX_IT,
            "kernel": args.kernel, "permuted": permuted, "impl": "oracle/_ref (the reference compiled "
            "from /root/reference/proj/src)", "seconds": round(dt, 1)}
    np.savez_compressed(
        fixture_path(args.kernel), history=res.residual_history, iterations=res.iterations,
        converged=res.converged, spmv_calls=res.spmv_calls,
        matrix_sha256=digest(m.row_offsets, m.col_indices, m.values), b_sha256=digest(b),
        solution_sha256=digest(res.solution), solution_norm=float(np.linalg.norm(res.solution)),
        solution_idx=idx, solution_samples=xs, meta=json.dumps(meta))
    print("wrote", fixture_path(args.kernel), flush=True)


if __name__ == "__main__":
    main()

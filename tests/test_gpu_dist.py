"""Row-partitioned SpMV and CG on one B200.

The in-process transport runs G partitions on the same device with the same
partition plan, halo exchange and rank-ordered dot products as the NCCL
transport, so the whole partitioned algorithm is checked here on 1 GPU:
SpMV bitwise against the single-GPU kernel (per-row sums are unchanged by
partitioning), CG histories within the reference comparator. The NCCL
transport itself is exercised with a 1-rank communicator (both
constructors); tests/test_dist_gloo.py covers the multi-rank protocol on CPU.
"""
import os

import numpy as np
import pytest

from tests.gpu_helpers import bits

pytestmark = pytest.mark.gpu


def same_up_to_zero_sign(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    both_zero = (a == 0) & (b == 0)
    return bool(np.all(both_zero | (bits(a) == bits(b))))


def hist_ok(got, want):
    got, want = np.asarray(got), np.asarray(want)
    return got.size == want.size and bool(np.all(np.abs(got - want) <= 1e-10 * (1.0 + want)))


@pytest.fixture(scope="module")
def fem():
    from paper_1501_00324_b200 import workloads as W
    from oracle.oracle import Csr

    n, _, ro, ci, v = W.elasticity_box(7, 6, 9)
    return Csr.make(n, n, ro, ci, v)


def test_partition_rule(ew, fem):
    b = ew.partition_rows(fem.row_offsets, 4)
    assert b[0] == 0 and b[-1] == fem.nrows and np.all(np.diff(b) >= 0)
    nnz = fem.row_offsets[-1]
    for g in range(1, 4):  # first row whose nnz prefix reaches g * nnz / G
        assert fem.row_offsets[b[g]] >= g * nnz // 4
        assert b[g] == 0 or fem.row_offsets[b[g] - 1] < g * nnz // 4


@pytest.mark.parametrize("nparts", [1, 2, 3, 5])
@pytest.mark.parametrize("kernel", ["k1", "k2", "csr_ref"])
def test_partitioned_spmv_matches_single_gpu(ew, R, fem, nparts, kernel):
    x = np.random.default_rng(nparts).uniform(0.1, 1.0, fem.ncols)
    a = ew.Csr(fem.nrows, fem.ncols, fem.row_offsets, fem.col_indices, fem.values)
    single = ew.Kernel(kernel, a, threshold=4).apply(x)
    d = ew.Dist.local(fem, nparts, kernel=kernel, threshold=4)
    assert d.owned == fem.nrows and d.nlocal == nparts
    y = d.spmv(x)
    if kernel == "k2":
        # a K2 row's chunk length is the max over the rows sharing its warp
        # (warp_layout.cpp:108-112), and partitioning regroups warps: the
        # summation association may differ, within the reference's 1e-12
        from tests.gpu_helpers import rel_close

        assert rel_close(y, single, 1e-12)
    else:
        assert same_up_to_zero_sign(y, single)
    if nparts > 1:
        assert sum(d.info(i)["nghost"] for i in range(nparts)) > 0


@pytest.fixture(scope="module")
def spd(F):
    # the reference's own SPD family for CG tests (test_solver.cpp:83)
    return F.fem_tet_graph(3000, 5, 21, 12)


@pytest.mark.parametrize("nparts", [1, 2, 4])
def test_partitioned_cg_matches_reference(ew, R, spd, nparts):
    b = R.spmv_csr(spd, np.ones(spd.ncols))
    diag = R.extract_diagonal(spd)
    ref = R.cg_csr(spd, b)
    d = ew.Dist.local(spd, nparts)
    res = d.cg_solve(b, diag)
    assert res.converged and res.iterations == ref.iterations and res.spmv_calls == ref.spmv_calls
    assert hist_ok(res.residual_history, ref.residual_history)
    assert np.allclose(res.solution, ref.solution, rtol=1e-8, atol=1e-10)


def test_partitioned_cg_ill_conditioned_fem(ew, R, fem):
    """Elasticity with a 1e-3 mass shift (kappa ~1e6): 145 iterations amplify
    summation-order rounding beyond 1e-10, for the single-GPU solver too; the
    partitioned run tracks the single-GPU device run as closely as that one
    tracks the sequential reference."""
    b = R.spmv_csr(fem, np.ones(fem.ncols))
    diag = R.extract_diagonal(fem)
    ref = R.cg_csr(fem, b)
    a = ew.Csr(fem.nrows, fem.ncols, fem.row_offsets, fem.col_indices, fem.values)
    one = ew.Kernel("k1", a).cg_solve(b, diag)
    part = ew.Dist.local(fem, 3).cg_solve(b, diag)
    assert one.iterations == ref.iterations == part.iterations
    drift_one = np.max(np.abs(one.residual_history - ref.residual_history) / (1 + ref.residual_history))
    drift_part = np.max(np.abs(part.residual_history - ref.residual_history) / (1 + ref.residual_history))
    assert drift_one < 1e-6 and drift_part < 1e-6


def test_partitioned_cg_long_run_and_errors(ew, R, spd):
    rng = np.random.default_rng(3)
    b = rng.uniform(-1, 1, spd.nrows)
    diag = R.extract_diagonal(spd)
    ref = R.cg_csr(spd, b, tol=1e-300, max_iterations=120, recompute=7)
    d = ew.Dist.local(spd, 3)
    res = d.cg_solve(b, diag, tol=1e-300, max_iterations=120, recompute_interval=7)
    assert res.iterations == 120 and not res.converged and res.spmv_calls == ref.spmv_calls
    assert hist_ok(res.residual_history, ref.residual_history)
    bad = b.copy()
    bad[-1] = np.inf
    with pytest.raises(ew.CgDivergenceError):
        d.cg_solve(bad, diag)
    zd = diag.copy()
    zd[0] = 0.0
    with pytest.raises(ValueError):
        d.cg_solve(b, zd)
    with pytest.raises(ValueError):
        ew.Dist.local(spd, 2, kernel="k1rs")


def _nccl_world1():
    import torch.distributed as dist

    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        dist.init_process_group("gloo", rank=0, world_size=1)


def test_nccl_transport_one_rank(ew, R, fem):
    """The NCCL code path with a 1-rank communicator: global and block
    constructors, SpMV and CG."""
    import torch  # noqa: F401  (loads libnccl into the process)
    import torch.distributed  # noqa: F401

    _nccl_world1()
    x = np.random.default_rng(9).uniform(0.1, 1.0, fem.ncols)
    a = ew.Csr(fem.nrows, fem.ncols, fem.row_offsets, fem.col_indices, fem.values)
    single = ew.Kernel("k1", a).apply(x)
    d = ew.Dist.nccl(fem, 1, 0, ew.nccl_unique_id())
    assert same_up_to_zero_sign(d.spmv(x), single)
    bounds = np.array([0, fem.nrows], np.int64)
    d2 = ew.Dist.block(fem.nrows, fem.row_offsets, fem.col_indices, fem.values, bounds, 0, ew.nccl_unique_id())
    assert same_up_to_zero_sign(d2.spmv(x), single)
    a_one = ew.Kernel("k1", a)
    b = R.spmv_csr(fem, np.ones(fem.ncols))
    one = a_one.cg_solve(b, R.extract_diagonal(fem))
    res = d2.cg_solve(b, R.extract_diagonal(fem))
    # one partition: same kernels, same reductions -> the single-GPU history
    assert res.iterations == one.iterations
    assert np.max(np.abs(res.residual_history - one.residual_history) / (1 + one.residual_history)) < 1e-6

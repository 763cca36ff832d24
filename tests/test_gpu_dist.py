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


@pytest.mark.parametrize("transport", ["copy", "peer"])
@pytest.mark.parametrize("nparts", [1, 2, 3, 5])
@pytest.mark.parametrize("kernel", ["k1", "k2", "csr_ref"])
def test_partitioned_spmv_matches_single_gpu(ew, R, fem, nparts, kernel, transport):
    x = np.random.default_rng(nparts).uniform(0.1, 1.0, fem.ncols)
    a = ew.Csr(fem.nrows, fem.ncols, fem.row_offsets, fem.col_indices, fem.values)
    single = ew.Kernel(kernel, a, threshold=4).apply(x)
    d = ew.Dist.local(fem, nparts, kernel=kernel, threshold=4, transport=transport)
    assert d.owned == fem.nrows and d.nlocal == nparts
    y = d.spmv(x)
    for _ in range(3):  # back-to-back exchanges: the peer transport's acks
        y2 = d.spmv(x)
        assert np.array_equal(bits(y2), bits(y))
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


@pytest.mark.parametrize("transport", ["copy", "peer"])
@pytest.mark.parametrize("nparts", [1, 2, 4])
def test_partitioned_cg_matches_reference(ew, R, spd, nparts, transport):
    b = R.spmv_csr(spd, np.ones(spd.ncols))
    diag = R.extract_diagonal(spd)
    ref = R.cg_csr(spd, b)
    d = ew.Dist.local(spd, nparts, transport=transport)
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


@pytest.mark.parametrize("transport", ["copy", "peer"])
def test_partitioned_cg_long_run_and_errors(ew, R, spd, transport):
    rng = np.random.default_rng(3)
    b = rng.uniform(-1, 1, spd.nrows)
    diag = R.extract_diagonal(spd)
    ref = R.cg_csr(spd, b, tol=1e-300, max_iterations=120, recompute=7)
    d = ew.Dist.local(spd, 3, transport=transport)
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


def _ipc_worker(rank, world, port, q):
    """One rank of the IPC transport; both ranks share the one GPU (CUDA IPC
    works between processes on the same device), so the push / mailbox
    protocol runs across real process boundaries.

    Two processes on one GPU (no MPS here) time-slice it: a rank's kernel
    spinning on a peer mailbox can keep the GPU until the 30 s peer timeout
    (the attempt then fails with a peer timeout, never with a silently wrong
    result: a timed-out operator reports it). So each attempt builds fresh
    operators, and the ranks agree on a retry (up to 4 attempts) when any
    rank saw a peer timeout; a wrong result without one fails at once. On
    one GPU per process (the real layout) there is no time-slicing."""
    try:
        import torch
        import torch.distributed as dist

        from oracle.oracle import Csr, Restatement
        from paper_1501_00324_b200 import capi
        from paper_1501_00324_b200 import workloads as W

        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        n, _, ro, ci, v = W.elasticity_box(6, 5, 7)
        m = Csr.make(n, n, ro, ci, v)
        R = Restatement()
        bounds = capi.partition_rows(ro, world)
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        bro = ro[r0:r1 + 1] - ro[r0]
        x = np.random.default_rng(5).uniform(0.1, 1.0, n)
        a = capi.Csr(n, n, ro, ci, v)
        single = capi.Kernel("k1", a).apply(x)
        sp = W.laplacian_box(9, 8, 7)
        n2, _, ro2, ci2, v2 = sp
        m2 = Csr.make(n2, n2, ro2, ci2, v2)
        b2 = R.spmv_csr(m2, np.ones(n2))
        ref = R.cg_csr(m2, b2)
        bounds2 = capi.partition_rows(ro2, world)
        s0, s1 = int(bounds2[rank]), int(bounds2[rank + 1])
        diag = R.extract_diagonal(m2)
        attempts = []
        for attempt in range(4):
            timed_out, err = 0, None
            ys, res = [], None
            try:
                d = capi.Dist.block_ipc(n, bro, ci[ro[r0]:ro[r1]], v[ro[r0]:ro[r1]], bounds, rank)
                d2 = capi.Dist.block_ipc(n2, ro2[s0:s1 + 1] - ro2[s0], ci2[ro2[s0]:ro2[s1]], v2[ro2[s0]:ro2[s1]],
                                         bounds2, rank)
                torch.cuda.synchronize()
                dist.barrier()
                ys = [d.spmv(x[r0:r1]) for _ in range(4)]
                torch.cuda.synchronize()
                dist.barrier()
                res = d2.cg_solve(b2[s0:s1], diag[s0:s1])
            except (capi.DeviceError, capi.CgDivergenceError) as e:
                timed_out, err = 1, repr(e)
            flags = [None] * world
            dist.all_gather_object(flags, timed_out)
            dist.barrier()
            d = d2 = None
            torch.cuda.synchronize()
            dist.barrier()
            attempts.append(err)
            if not any(flags):
                break
        if res is None or any(flags):
            raise RuntimeError(f"peer timeouts on every attempt (time-sliced GPU): {attempts}")
        ok_spmv = all(same_up_to_zero_sign(y, single[r0:r1]) for y in ys)
        ok_cg = (res.converged and res.iterations == ref.iterations and
                 hist_ok(res.residual_history, ref.residual_history) and
                 np.allclose(res.solution, ref.solution[s0:s1], rtol=1e-8, atol=1e-10))
        detail = {"spmv_bad_calls": [i for i, y in enumerate(ys) if not same_up_to_zero_sign(y, single[r0:r1])],
                  "converged": res.converged, "it": res.iterations, "ref_it": ref.iterations,
                  "hist_ok": hist_ok(res.residual_history, ref.residual_history), "attempts": attempts}
        q.put((rank, ok_spmv, ok_cg, detail, ref.iterations))
        dist.destroy_process_group()
    except Exception as e:  # reported to the parent
        q.put((rank, False, False, repr(e), None))


def test_ipc_transport_two_processes(ew, tmp_path):
    """Two processes, one partition each, over the CUDA IPC peer transport
    (gloo only for the setup allgather), run concurrently on this GPU under a
    private MPS daemon when the image has one (else time-sliced, with the
    worker's retries)."""
    import multiprocessing as mp
    import socket

    from tests.gpu_helpers import mps_environment

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with mps_environment(tmp_path) as env:
        saved = dict(os.environ)
        if env:  # spawned children take the environment at start
            os.environ.update(env)
        try:
            procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
            for p in procs:
                p.start()
        finally:
            os.environ.clear()
            os.environ.update(saved)
        out = [q.get(timeout=600) for _ in procs]
        for p in procs:
            p.join(timeout=60)
    for rank, ok_spmv, ok_cg, it, ref_it in sorted(out, key=lambda t: t[0]):
        print("rank", rank, "mps" if env else "time-sliced", it)
        assert ok_spmv, (rank, it)
        assert ok_cg, (rank, it)


def test_bench_two_ranks_functional(tmp_path):
    """bench.py's N > 1 path (partitioned SpMV + CG, IPC transport) under
    torchrun with two ranks sharing this GPU (concurrently under a private
    MPS daemon when available): runs end to end and prints one JSON line with
    both metrics (a functional check, not a measurement)."""
    import json
    import socket
    import subprocess
    import sys

    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    from tests.gpu_helpers import mps_environment

    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2", "--steps", "5", "--warmup", "3",
           "--scale", "0.25", "--iterations", "60", "--cg-steps", "1", "--no-cpu-baseline"]
    with mps_environment(tmp_path) as mps:
        env = dict(mps or os.environ, EW_BENCH_SHARE_GPU="1")
        out = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["config"]["transport"] == "ipc"
    assert line["cg"]["n_gpus"] == 2 and line["cg"]["value"] > 0
    assert line["cg"]["config"]["final_residual"] < 1.0


def test_bench_one_gpu_all_lines():
    """bench.py at N=1 on scaled-down configs: the SpMV headline plus the
    config-4 CG line in both row orders and the partitioned config-5 CG
    line (strong-scaling path with one rank), every timed solve at full
    length."""
    import json
    import subprocess
    import sys

    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "bench.py", "--steps", "5", "--warmup", "3", "--scale", "0.15", "--iterations", "60",
           "--cg-steps", "2", "--no-cpu-baseline"]
    out = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 1 and line["value"] > 0 and line["e2e"]["value"] > 0
    c4 = line["cg_c4"]
    assert c4["value"] > 0 and c4["config"]["row_order"] == "locality"
    assert c4["config"]["iterations_run"] == [60, 60]
    assert c4["reference_row_order"]["value"] > 0
    c5 = line["cg"]
    assert c5["scaling"] == "strong" and c5["config"]["config"] == "c5" and c5["value"] > 0
    assert c5["config"]["iterations_run"] == [60, 60]


@pytest.mark.parametrize("ngpus", [1, 2, 4])
def test_mgpu_single_process_matches_partitioned(ew, R, ngpus):
    """ew_mgpu_* (one process, one host thread + stream per block, peers
    over peer access) with every block mapped onto this GPU: the same
    partitions, kernels and rank-ordered sums as the in-process peer
    transport, so SpMV bitwise the single-GPU K1 and the CG history, count
    and solution bitwise those of Dist.local(..., transport="peer")."""
    from oracle.oracle import Csr
    from paper_1501_00324_b200 import workloads as W

    n, _, ro, ci, v = W.elasticity_box(14, 13, 12)
    m = Csr.make(n, n, ro, ci, v)
    mg = ew.Mgpu(m, ngpus, devices=[0] * ngpus)
    x = np.random.default_rng(7).uniform(-1, 1, n)
    single = ew.Kernel("k1", ew.Csr(n, n, ro, ci, v)).apply(x)
    y = mg.spmv(x)
    both_zero = (y == 0) & (single == 0)
    assert np.all(both_zero | (y.view(np.int64) == single.view(np.int64)))
    b = R.spmv_csr(m, np.ones(n))
    diag = R.extract_diagonal(m)
    res = mg.cg_solve(b, diag, tol=1e-10, max_iterations=2000)
    want = ew.Dist.local(m, ngpus, transport="peer" if ngpus > 1 else "copy").cg_solve(b, diag, tol=1e-10,
                                                                                      max_iterations=2000)
    assert res.converged and res.iterations == want.iterations
    assert res.spmv_calls == 1 + res.iterations + res.iterations // 50
    assert np.array_equal(res.residual_history.view(np.int64), want.residual_history.view(np.int64))
    assert np.array_equal(res.solution.view(np.int64), want.solution.view(np.int64))
    # against the reference (sequential dot products): the comparator
    # (test_solver.cpp:104-112) until CG's amplification of rounding
    # differences takes over (~200 iterations on these elasticity operators,
    # as for the reference's own permuted-vs-plain pair), 1e-8 after
    ref = R.cg_csr(m, b, tol=1e-10, max_iterations=2000)
    assert res.iterations == ref.iterations
    dev = np.abs(res.residual_history - ref.residual_history) / (1 + ref.residual_history)
    assert np.all(dev[:150] <= 1e-10) and np.all(dev <= 1e-8)
    assert np.max(np.abs(res.solution - ref.solution)) <= 1e-9


def test_mgpu_errors(ew):
    from oracle.oracle import Csr

    m = Csr.make(3, 3, [0, 1, 2, 3], [0, 1, 5], [1.0, 1.0, 1.0])
    with pytest.raises(ValueError):
        ew.Mgpu(m, 1, devices=[0])  # column out of range
    m = Csr.make(3, 3, [0, 1, 2, 3], [0, 1, 2], [1.0, 1.0, 1.0])
    with pytest.raises(ValueError):
        ew.Mgpu(m, 2, devices=[0, 99])  # no such device
    with pytest.raises(ValueError):
        ew.Mgpu(m, 1, devices=[0], kernel="k1rs")


def test_reference_api_multi_gpu_cg(ew):
    """The reference's Python entry (_ellwarp.cg_solve, module.cpp:227-249)
    with the addition ngpus / devices: the row-partitioned solve from one
    process (every block on this GPU here); same dict as the reference, the
    single-GPU iteration count."""
    from paper_1501_00324_b200 import load_ellwarp

    e = load_ellwarp()
    m = e.laplacian3d(12, 11, 10)
    b = e.spmv_reference(m, [1.0] * m.nrows)
    one = e.cg_solve(m, b, kernel="k1", tol=1e-8)
    two = e.cg_solve(m, b, kernel="k1", tol=1e-8, devices=[0, 0, 0])
    assert one["converged"] and two["converged"]
    assert two["iterations"] == one["iterations"]
    assert two["spmv_calls"] == one["spmv_calls"]
    assert np.allclose(two["solution"], 1.0, atol=1e-6)


def test_dist_layout_bytes(ew):
    """ew_dist_get_layout_bytes: one partition holds the single-GPU K1
    layout (same slots, same streamed bytes); split partitions count their
    interior and boundary layouts, every entry stored once."""
    from oracle.oracle import Csr
    from paper_1501_00324_b200 import workloads as W

    n, _, ro, ci, v = W.elasticity_box(9, 8, 7)
    m = Csr.make(n, n, ro, ci, v)
    ki = ew.Kernel("k1", ew.Csr(n, n, ro, ci, v)).info()
    one = ew.Dist.local(m, 1, transport="copy").info(0)
    assert one["stored_slots"] == ki.stored_slots
    assert one["stream_bytes"] == 8 * ki.stored_slots + ki.col_stream_bytes
    d = ew.Dist.local(m, 3, transport="peer")
    parts = [d.info(i) for i in range(3)]
    assert sum(p["stored_slots"] for p in parts) >= m.nnz
    for p in parts:
        assert 10 * p["stored_slots"] <= p["stream_bytes"] <= 12 * p["stored_slots"]

"""The N>1 protocol of the row-partitioned operator on CPU (world_size 2,
torch.distributed gloo), mirroring ew_dist.cu message for message: the
library's nnz-balanced partition rule (ew_partition_rows, host function),
ghost lists grouped by owner, ghost-request exchange (counts all-gathered,
ids point-to-point), halo exchange per SpMV, partition totals all-gathered
and summed in rank order. Results are checked against the C oracle."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, queue):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from oracle.oracle import Reference
    from paper_1501_00324_b200 import capi

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    F = Reference()
    m = F.fem_tet_graph(2000, 5, 21, 12)
    bounds = capi.partition_rows(m.row_offsets, world)
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    nloc = r1 - r0
    ro = m.row_offsets[r0:r1 + 1] - m.row_offsets[r0]
    ci = m.col_indices[m.row_offsets[r0]:m.row_offsets[r1]]
    v = m.values[m.row_offsets[r0]:m.row_offsets[r1]]
    owner = lambda c: int(np.searchsorted(bounds, c, side="right") - 1)  # noqa: E731
    ghosts = np.unique(ci[(ci < r0) | (ci >= r1)])
    my_need = np.zeros(world, np.int64)
    for c in ghosts:
        my_need[owner(c)] += 1
    # setup exchange: counts all-gathered, ghost ids point to point
    all_need = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(all_need, torch.from_numpy(my_need))
    goff = np.concatenate([[0], np.cumsum(my_need)])
    sends, recvs = {}, {}
    reqs = []
    for h in range(world):
        if h == rank:
            continue
        if my_need[h]:
            reqs.append(dist.isend(torch.from_numpy(ghosts[goff[h]:goff[h + 1]].copy()), h))
        cnt = int(all_need[h][rank])
        if cnt:
            recvs[h] = torch.zeros(cnt, dtype=torch.int64)
            reqs.append(dist.irecv(recvs[h], h))
    for r in reqs:
        r.wait()
    send_lists = {h: t.numpy() - r0 for h, t in recvs.items()}
    lci = np.where((ci >= r0) & (ci < r1), ci - r0, nloc + np.searchsorted(ghosts, ci))
    recv_off = np.concatenate([[0], np.cumsum([int(my_need[h]) if h != rank else 0 for h in range(world)])])

    def halo(xo):
        ext = np.concatenate([xo, np.zeros(len(ghosts))])
        reqs = []
        bufs = {}
        for h in range(world):
            if h == rank:
                continue
            if h in send_lists:
                reqs.append(dist.isend(torch.from_numpy(xo[send_lists[h]].copy()), h))
            if my_need[h]:
                bufs[h] = torch.zeros(int(my_need[h]), dtype=torch.float64)
                reqs.append(dist.irecv(bufs[h], h))
        for r in reqs:
            r.wait()
        for h, t in bufs.items():
            ext[nloc + recv_off[h]:nloc + recv_off[h + 1]] = t.numpy()
        return ext

    def spmv(xo):
        ext = halo(xo)
        y = np.zeros(nloc)
        for r in range(nloc):
            s = 0.0
            for k in range(ro[r], ro[r + 1]):
                s += v[k] * ext[lci[k]]
            y[r] = s
        return y

    def gdot(a, b):  # partition totals all-gathered, summed in rank order
        parts = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.tensor([float(np.dot(a, b))], dtype=torch.float64))
        t = 0.0
        for p in parts:
            t += float(p[0])
        return t

    x_glob = np.linspace(0.1, 1.0, m.ncols)
    y_loc = spmv(x_glob[r0:r1])
    # Jacobi PCG (cg.cpp:25-104) with the same reductions as the device solver
    b = np.ones(nloc) * 0.0 + (F.spmv_csr(m, np.ones(m.ncols))[r0:r1])
    diag = F.extract_diagonal(m)[r0:r1]
    bnorm = np.sqrt(gdot(b, b))
    xs = np.zeros(nloc)
    r = b - spmv(xs)
    hist = [np.sqrt(gdot(r, r)) / bnorm]
    z = r / diag
    p = z.copy()
    rz = gdot(r, z)
    its = 0
    for k in range(1, 1001):
        q = spmv(p)
        alpha = rz / gdot(p, q)
        xs += alpha * p
        r -= alpha * q
        if k % 50 == 0:
            r = b - spmv(xs)
        its = k
        rel = np.sqrt(gdot(r, r)) / bnorm
        hist.append(rel)
        if rel <= 1e-8:
            break
        z = r / diag
        rz_new = gdot(r, z)
        p = z + (rz_new / rz) * p
        rz = rz_new
    queue.put((rank, r0, y_loc, xs, hist, its, len(ghosts), sum(len(s) for s in send_lists.values())))
    dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_two_rank_partitioned_spmv_and_cg(R, F):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=540) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    m = F.fem_tet_graph(2000, 5, 21, 12)
    y = np.concatenate([o[2] for o in out])
    want = R.spmv_csr(m, np.linspace(0.1, 1.0, m.ncols))
    assert np.allclose(y, want, rtol=1e-12, atol=0)
    # halos are symmetric for a symmetric pattern: what 0 sends, 1 receives
    assert out[0][6] == out[1][7] and out[1][6] == out[0][7] and out[0][6] > 0
    ref = R.cg_csr(m, R.spmv_csr(m, np.ones(m.ncols)))
    hist = np.asarray(out[0][4])
    assert out[0][5] == out[1][5] == ref.iterations
    assert np.all(np.abs(hist - ref.residual_history) <= 1e-10 * (1 + ref.residual_history))
    xs = np.concatenate([o[3] for o in out])
    assert np.allclose(xs, ref.solution, rtol=1e-8, atol=1e-10)


def _plan_worker(rank, world, port, queue):
    """One rank of the library's own IPC setup exchange (ew_dist_plan_block:
    ghost list, counts all-gathered, ghost ids all-gathered, per-peer send
    lists) over torch.distributed gloo: the code ew_dist_create_block_ipc
    runs before any device work."""
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from oracle.oracle import Reference
    from paper_1501_00324_b200 import capi

    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        m = Reference().fem_tet_graph(3000, 5, 21, 12)
        bounds = capi.partition_rows(m.row_offsets, world)
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        ro = m.row_offsets[r0:r1 + 1] - m.row_offsets[r0]
        ci = m.col_indices[m.row_offsets[r0]:m.row_offsets[r1]]
        ghosts, sends = capi.dist_plan_block(ro, ci, bounds, rank)
        queue.put((rank, bounds.tolist(), ghosts.tolist(), [s.tolist() for s in sends]))
        dist.destroy_process_group()
    except Exception as e:  # reported to the parent
        queue.put((rank, None, repr(e), None))


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [2, 3])
def test_library_ipc_setup_exchange(F, world):
    """ew_dist_plan_block from `world` processes (gloo allgather): every
    rank's ghost list is the ascending set of its block's columns outside
    the block, and what rank g sends to h is exactly the part of h's ghost
    list that g owns."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_plan_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=240) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(60)
    for o in out:
        assert o[1] is not None, o[2]
    m = F.fem_tet_graph(3000, 5, 21, 12)
    bounds = np.asarray(out[0][1])
    for g in range(world):
        r0, r1 = bounds[g], bounds[g + 1]
        cols = m.col_indices[m.row_offsets[r0]:m.row_offsets[r1]]
        want = np.unique(cols[(cols < r0) | (cols >= r1)])
        assert np.array_equal(np.asarray(out[g][2], np.int64), want)
    for g in range(world):
        for h in range(world):
            gh = np.asarray(out[h][2], np.int64)
            owned = gh[(gh >= bounds[g]) & (gh < bounds[g + 1])] if h != g else np.zeros(0, np.int64)
            assert np.array_equal(np.asarray(out[g][3][h], np.int64), owned), (g, h)
    assert sum(len(s) for o in out for s in o[3]) > 0

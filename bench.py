"""B200 bench for the ELL-WARP SpMV + Jacobi PCG path (BASELINE.json).

Default (N=1): fp64 SpMV effective bandwidth on config 2 (3-DOF linear
elasticity tet mesh, 1,975,509 rows, 87.3M nonzeros) through the prepared
K1 kernel, device-resident inputs. One JSON line on stdout (rank 0).

  value      paper-effective bandwidth 20*nnz / t (csr.cpp:92)
  roofline   algorithmic bytes 12*nnz + 8*nrows + 8*ncols of the dominant
             kernel (k1_kernel) / its CUDA-event time vs MEASURED_PEAKS hbm
  e2e        same metric through ew_kernel_apply with pinned HOST buffers,
             H2D x + D2H y inside the timed region
  cpu_baseline  the reference's own prepare_kernel("k1").apply, compiled
             from its sources (oracle/_ref), single thread, on this host

--workload cg: Jacobi PCG iterations/s on config 4 (ventricle-like mesh,
5M rows, random renumbering), k1rs in permuted space, 1000 iterations.

--impl reference: the reference's CPU implementation on the same config and
metric (oracle/_ref, 1 thread: the reference has no threading).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c1": dict(name="fp64 SpMV, 3D linear-tet Laplacian 64^3 nodes (262,144 rows)", gen="laplacian_box",
               dims=(63, 63, 63)),
    "c2": dict(name="fp64 SpMV, 3-DOF linear-elasticity tet mesh 87^3 nodes (1,975,509 rows)",
               gen="elasticity_box", dims=(86, 86, 86)),
    "c4": dict(name="Jacobi PCG 1000 it, jittered+renumbered tet ventricle-like mesh 171^3 nodes (5,000,211 rows)",
               gen="ventricle_box", dims=(170, 170, 170)),
    # config 5 whole on one GPU through a plain prepared kernel (SpMV / CG)
    "c5full": dict(name="fp64 3-DOF linear-elasticity tet mesh 322^3 nodes (100,158,744 rows), one GPU",
                   gen="elasticity_box_slabbed", dims=(321, 321, 321)),
}
# config 5 for the partitioned CG: the same 100,158,744-row mesh at every N,
# rank r generating only its z-slab of node layers (strong scaling)
C5_DIMS = (321, 321, 321)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(key):
    """DRAM bytes per launch of the dominant kernel from a committed ncu
    capture (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f)[key]["traffic_bytes_per_launch"]
    except Exception:  # noqa: BLE001
        return None


def build_matrix(cfg_key, scale=1.0):
    from paper_1501_00324_b200 import workloads as W

    c = CONFIGS[cfg_key]
    dims = tuple(max(2, int(round(d * scale))) for d in c["dims"])
    t = time.time()
    n, nc, ro, ci, v = getattr(W, c["gen"])(*dims)
    log(f"[bench] {cfg_key} {dims}: {n} rows, {ro[-1]} nnz, generated in {time.time() - t:.1f}s")
    return n, nc, ro, ci, v


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        if os.environ.get("EW_BENCH_NO_CLOCKS") == "1":  # diagnosis only: no sampler
            return self
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            t = time.time()
            # sampler live (and past its first queries, which can stall the
            # GPU for tens of ms) before timing starts
            while len(self.rows) < 6 and time.time() - t < 5.0:
                time.sleep(0.01)
            self.rows.clear()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([s.strip() for s in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:  # noqa: BLE001
                self.proc.kill()
            self.thread.join(1)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for nm, val in zip(names, r[4:8]):
                    if val.strip().lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_init(n_gpus):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        if os.environ.get("EW_BENCH_SHARE_GPU"):
            # functional runs of the N > 1 path on a box with fewer GPUs than
            # ranks (ranks share devices; the IPC transport works between
            # processes on one device; gloo for the setup allgather). Not a
            # measurement.
            local = local % torch.cuda.device_count()
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(v, world):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64, device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(vals, world):
    if world == 1:
        return [float(x) for x in vals]
    import torch
    import torch.distributed as dist

    t = torch.tensor(vals, dtype=torch.float64, device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t)
    return [float(x) for x in t.tolist()]


# ---------------------------------------------------------------------------
# CPU: the reference (oracle/_ref) on a bounded sample
# ---------------------------------------------------------------------------
def reference_spmv_rate(n, nc, ro, ci, v, kernel="k1", budget_s=15.0, max_calls=50, warmup=1):
    from oracle.oracle import Csr, Reference

    F = Reference()
    m = Csr.make(n, nc, ro, ci, v)
    x = np.random.default_rng(1).uniform(0.1, 1.0, nc)
    y = np.empty(n)
    t0 = time.perf_counter()
    h = F.prepare(kernel, m)
    t_prep = time.perf_counter() - t0
    for _ in range(warmup):
        F.run(h, x, y)
    times = []
    t_start = time.perf_counter()
    while len(times) < max_calls and (time.perf_counter() - t_start) < budget_s:
        t = time.perf_counter()
        F.run(h, x, y)
        times.append(time.perf_counter() - t)
    F.free_prepared(h)
    med = float(np.median(times))
    return med, len(times), t_prep


def port_spmv_rate_mt(n, nc, ro, ci, v, threads, budget_s=8.0, max_calls=50):
    """The oracle's row-parallel (pthreads) CSR SpMV port on `threads` host
    threads: a multi-core CPU comparison beside the single-threaded
    reference (same row sums)."""
    from oracle.oracle import Csr, Restatement

    R = Restatement()
    m = Csr.make(n, nc, ro, ci, v)
    x = np.random.default_rng(1).uniform(0.1, 1.0, nc)
    y = np.empty(n)
    R.spmv_csr_mt(m, x, threads, y)  # warm-up
    times = []
    t_start = time.perf_counter()
    while len(times) < max_calls and (time.perf_counter() - t_start) < budget_s:
        t = time.perf_counter()
        R.spmv_csr_mt(m, x, threads, y)
        times.append(time.perf_counter() - t)
    return float(np.median(times)), len(times)


def reference_cg_rate(n, nc, ro, ci, v, iters):
    from oracle.oracle import Csr, Reference

    F = Reference()
    m = Csr.make(n, nc, ro, ci, v)
    b = F.spmv_csr(m, np.ones(nc))
    t = time.perf_counter()
    res = F.cg("csr_ref", m, b, tol=1e-300, max_iterations=iters)
    dt = time.perf_counter() - t
    return res.iterations / dt, res.iterations, dt


# ---------------------------------------------------------------------------
# multi-GPU: one z-slab row block of the elasticity box per rank
# ---------------------------------------------------------------------------
def build_slab(args, rank, world):
    """Rank `rank`'s rows of a box(86, 86, 87*world - 1) elasticity mesh: every
    rank owns 87 node layers, i.e. a config-2-sized block (weak scaling)."""
    from paper_1501_00324_b200 import workloads as W

    nx = ny = max(2, int(round(86 * args.scale)))
    per = nx + 1
    nz = per * world - 1
    layers = W.slab_layers(nz, world)
    t = time.time()
    rb, ng, ro, ci, v = W.box_rows("elasticity", nx, ny, nz, layers[rank], layers[rank + 1])
    bounds = np.array([3 * (nx + 1) * (ny + 1) * k for k in layers], np.int64)
    log(f"[bench] rank {rank}: slab layers [{layers[rank]}, {layers[rank + 1]}) of box({nx},{ny},{nz}): "
        f"{ro.size - 1} rows, {ro[-1]} nnz, {time.time() - t:.1f}s")
    return ng, ro, ci, v, bounds


def build_c5_block(args, rank, world):
    """Rank `rank`'s rows of config 5 (box(321, 321, 321), 3-DOF elasticity,
    100,158,744 rows): node layers slab_layers(321, world)[rank:rank + 2],
    generated slab by slab on host threads (strong scaling: the global mesh
    is the same at every N)."""
    from paper_1501_00324_b200 import workloads as W

    nx, ny, nz = (max(2, int(round(d * args.scale))) for d in C5_DIMS)
    layers = W.slab_layers(nz, world)
    t = time.time()
    workers = max(1, min(16, (os.cpu_count() or 8) // world))
    rb, ng, ro, ci, v = W.box_rows_slabbed("elasticity", nx, ny, nz, layers[rank], layers[rank + 1],
                                           workers=workers)
    bounds = np.array([3 * (nx + 1) * (ny + 1) * k for k in layers], np.int64)
    log(f"[bench] rank {rank}: config-5 layers [{layers[rank]}, {layers[rank + 1]}) of box({nx},{ny},{nz}): "
        f"{ro.size - 1} rows, {ro[-1]} nnz, {time.time() - t:.1f}s ({workers} threads)")
    return ng, ro, ci, v, bounds


def step_times(ev0, marks):
    """Per-step device times (ms) from the start event and one event per step."""
    out, prev = [], ev0
    for m in marks:
        out.append(prev.elapsed_time(m))
        prev = m
    return out


def dist_operator(args, rank, world, shape="c2-slab"):
    """This rank's partition of the slab operator ("c2-slab": a config-2-sized
    block per GPU; "c5": its share of config 5). Transport "ipc" (default):
    CUDA IPC peer stores + mailboxes over NVLink, no NCCL on the data path;
    "nccl": ncclSend/Recv halos and ncclAllGather dots."""
    import torch.distributed as dist

    from paper_1501_00324_b200 import capi

    ng, ro, ci, v, bounds = build_c5_block(args, rank, world) if shape == "c5" else build_slab(args, rank, world)
    kid = args.kernel if args.kernel in ("k1", "k2", "csr_ref") else "k1"
    t = time.time()
    transport = args.transport
    d = None
    if transport == "ipc":
        try:
            d = capi.Dist.block_ipc(ng, ro, ci, v, bounds, rank, kernel=kid)
        except (capi.DeviceError, ValueError) as e:
            log(f"[bench] rank {rank}: IPC transport unavailable ({e}); falling back to NCCL")
            transport = "nccl"
    if d is None:
        obj = [capi.nccl_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(obj, src=0)
        d = capi.Dist.block(ng, ro, ci, v, bounds, rank, obj[0], kernel=kid)
    args.transport_used = transport
    info = d.info()
    log(f"[bench] rank {rank}: partitioned operator ({transport}) in {time.time() - t:.2f}s, {info['nghost']} ghosts, "
        f"{info['nsend']} sent per exchange")
    info["bounds"] = bounds
    return d, ng, ro, ci, v, info


# ---------------------------------------------------------------------------
# GPU arms
# ---------------------------------------------------------------------------
def k1_label(k, info):
    """Which K1 kernel form layout_spmv launches for this layout (ew_spmv.cu)."""
    slots, narrow = int(info.stored_slots), int(info.narrow_slots)
    grouped = info.col_stream_bytes < 2 * narrow + 4 * (slots - narrow)  # lanes share column lists
    g = ", grouped column lists" if grouped else ""
    if narrow:
        return f"k1_kernel (16-bit columns on narrow warps, compact_layout{g})"
    if slots * 12 > 64 << 20 and slots >= 24 * info.nrows:
        return f"k1_stream_kernel (grid-stride K1: layout beyond L2, >= 24 slots/row{g})"
    return f"k1_kernel{' (' + g[2:] + ')' if g else ''}"


def run_spmv(args, rank, world, local):
    if world > 1:
        return run_spmv_dist(args, rank, world, local)
    import torch

    from paper_1501_00324_b200 import capi

    hbm, peak_src = peaks()
    n, nc, ro, ci, v = build_matrix(args.config, args.scale)
    nnz = int(ro[-1])
    t = time.time()
    a = capi.Csr(n, nc, ro, ci, v)
    k = capi.Kernel(args.kernel, a, threshold=args.threshold, row_order=args.row_order)
    torch.cuda.synchronize()
    t_prepare = time.time() - t
    log(f"[bench] rank {rank}: upload+validate+prepare({args.kernel}) {t_prepare:.2f}s, "
        f"stored_slots {k.stored_slots} ({k.stored_slots - nnz} padded)")
    del a  # the prepared kernel keeps only its layout
    torch.cuda.empty_cache()
    x = torch.tensor(np.random.default_rng(1).uniform(0.1, 1.0, nc), device="cuda")
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()
    apply = k.apply_permuted if args.permuted else k.apply

    # warm-up, then exactly K timed steps between barriers + syncs
    for _ in range(args.warmup):
        apply(x, y, stream=stream)
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        # the timed loop is a few ms (shorter than one nvidia-smi sample):
        # the sampler records the clocks over a 0.5 s soak of the same
        # launches right before it, on the same stream, without a gap
        t_soak = time.perf_counter()
        while time.perf_counter() - t_soak < 0.5:
            for _ in range(50):
                apply(x, y, stream=stream)
            torch.cuda.current_stream().synchronize()
        l0 = capi.launch_count()
        ev0.record(stream)
        for _ in range(args.steps):
            apply(x, y, stream=stream)
        ev1.record(stream)
        torch.cuda.synchronize()
        launches = capi.launch_count() - l0
    barrier(world)
    ms_local = ev0.elapsed_time(ev1) / args.steps
    ms = max_over_ranks(ms_local, world)

    eff_bytes = 20 * nnz
    alg_bytes = 12 * nnz + 8 * n + 8 * nc
    value = world * eff_bytes / (ms * 1e-3) / 1e9
    # dominant kernel: one k1_kernel launch per step (gather kernels only for
    # r/rs apply); its per-launch time is the step time when launches == steps
    kern_ms = ms_local if launches == args.steps else None
    achieved = alg_bytes / (kern_ms * 1e-3) / 1e9 if kern_ms else None
    # the bytes the layout actually streams: 16-bit columns on the narrow
    # warps (compact_layout), int32 elsewhere, padding slots included
    kinfo = k.info()
    slots, narrow = int(kinfo.stored_slots), int(kinfo.narrow_slots)
    streamed = 8 * slots + int(kinfo.col_stream_bytes) + 8 * n + 8 * nc
    streamed_gbs = streamed / (kern_ms * 1e-3) / 1e9 if kern_ms else None

    # end-to-end through the C ABI with pinned host buffers
    xh = torch.empty(nc, dtype=torch.float64, pin_memory=True)
    xh.copy_(x.cpu())
    yh = torch.empty(n, dtype=torch.float64, pin_memory=True)
    xn, yn = xh.numpy(), yh.numpy()
    k_e2e = 200
    for _ in range(10):
        apply(xn, yn)
    barrier(world)
    calls = []
    t = time.perf_counter()
    for _ in range(k_e2e):
        t1 = time.perf_counter()
        apply(xn, yn)
        calls.append(time.perf_counter() - t1)
    e2e_ms = max_over_ranks((time.perf_counter() - t) * 1e3 / k_e2e, world)
    e2e_val = world * eff_bytes / (e2e_ms * 1e-3) / 1e9
    calls_ms = np.array(calls) * 1e3
    # this box's PCIe: the same bytes as one call's x upload and y download,
    # plain pinned copies (context for the e2e number, which is copy-bound)
    xg = torch.empty(nc, dtype=torch.float64, device="cuda")
    yg = torch.empty(n, dtype=torch.float64, device="cuda")
    pcie = {}
    for name, fn, nbytes in (("h2d", lambda: xg.copy_(xh, non_blocking=True), 8 * nc),
                             ("d2h", lambda: yh.copy_(yg, non_blocking=True), 8 * n)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(20):
            fn()
        torch.cuda.synchronize()
        pcie[f"{name}_gbs"] = round(nbytes * 20 / (time.perf_counter() - t) / 1e9, 1)
    # both directions at once on two streams (what the pipelined call needs):
    # the floor of one call is (x + y bytes) / this aggregate rate
    s_up, s_dn = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(20):
        with torch.cuda.stream(s_up):
            xg.copy_(xh, non_blocking=True)
        with torch.cuda.stream(s_dn):
            yh.copy_(yg, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    pcie["both_gbs"] = round((8 * nc + 8 * n) * 20 / dt / 1e9, 1)
    pcie["call_floor_ms"] = round(dt / 20 * 1e3, 4)
    del xg, yg

    out = {
        "metric": "SpMV effective GB/s (20 B/nnz, PAPER.md:553)",
        "value": round(value, 2),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 5),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded structured tet mesh, values from P1 elasticity element matrices)",
        "config": {"workload": CONFIGS[args.config]["name"], "config": args.config, "kernel": args.kernel,
                   "permuted": bool(args.permuted), "nrows": n, "nnz": nnz, "stored_slots": k.stored_slots,
                   "kernel_device_bytes": int(kinfo.device_bytes),
                   "per_rank": "independent copy per GPU" if world > 1 else "single GPU",
                   "l2": "inputs larger than L2 (%.2f GB algorithmic bytes vs 126 MB L2)" % (alg_bytes / 1e9)
                   if alg_bytes > 3 * 126e6 else "L2-resident working set: warm-L2 number"},
        "effective_pct_of_hbm": round(100 * value / world / hbm, 2),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1) if achieved else None, "peak": hbm,
                     "peak_source": peak_src, "unit": "GB/s",
                     "frac": round(achieved / hbm, 4) if achieved else None,
                     "traffic": ncu_traffic(f"{args.config}/{args.kernel}") if args.scale == 1.0 else None,
                     "traffic_source": "profiles/ncu_traffic.json (ncu dram__bytes_read+write per launch)",
                     "kernel": k1_label(k, kinfo) if args.kernel.startswith("k1") else "k2_kernel",
                     "algorithmic_bytes_per_launch": alg_bytes,
                     "streamed_bytes_per_launch": streamed,
                     "streamed_frac": round(streamed_gbs / hbm, 4) if streamed_gbs else None,
                     "note": "achieved/frac: the reference format's bytes (12 B/nnz + 8 n + 8 ncols, SURVEY 8d) "
                             "over the kernel time; streamed_frac: the bytes this layout moves (values, then "
                             "%.2f B of column per slot: 16-bit offsets on %.1f%% of the slots, lanes with equal "
                             "column lists sharing one) over the same time"
                             % (kinfo.col_stream_bytes / max(slots, 1), 100.0 * narrow / max(slots, 1))},
        "e2e": {"value": round(e2e_val, 2), "unit": "GB/s", "h2d_bytes_per_step": 8 * nc,
                "d2h_bytes_per_step": 8 * n, "ms_per_step": round(e2e_ms, 4),
                "call_ms_min_median_max": [round(float(calls_ms.min()), 4), round(float(np.median(calls_ms)), 4),
                                           round(float(calls_ms.max()), 4)],
                "path": "ew_kernel_apply(EW_MEM_HOST), pinned host x/y",
                "pcie_copy_gbs": dict(pcie, note="plain pinned copies of one call's x (H2D) and y (D2H) bytes on "
                                                 "this box: each direction alone, and both at once (call_floor_ms: "
                                                 "the copies of one call with nothing else to do)")},
        "gpu_launches": int(launches),
        "clocks": dict(clk.summary(), window="0.5 s soak of the same launches right before the timed loop + the "
                                              "timed loop"),
        "prepare_s": round(t_prepare, 3),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rows, what = n, f"full {args.config} matrix"
        if args.config == "c5full":
            # the reference's host copies of a 100M-row matrix would not fit
            # beside ours: a bounded sample, the first 2% of the rows
            rows = n // 50
            what = f"rows [0, {rows}) of {args.config} (all columns)"
        rnnz = int(ro[rows])
        med, calls, t_prep = reference_spmv_rate(rows, nc, ro[:rows + 1], ci[:rnnz], v[:rnnz], kernel=args.kernel)
        out["cpu_baseline"] = {"value": round(20 * rnnz / med / 1e9, 3), "unit": "GB/s", "cores": 1,
                               "kind": "reference",
                               "sample": f"{what}, median of {calls} prepare_kernel('"
                                         f"{args.kernel}').apply calls (oracle/_ref, 1 thread); "
                                         f"CPU layout build {t_prep:.1f}s"}
        threads = os.cpu_count() or 1
        mt, mcalls = port_spmv_rate_mt(rows, nc, ro[:rows + 1], ci[:rnnz], v[:rnnz], threads)
        out["cpu_baseline_multicore"] = {"value": round(20 * rnnz / mt / 1e9, 3), "unit": "GB/s", "cores": threads,
                                         "kind": "port",
                                         "sample": f"{what}, median of {mcalls} row-parallel CSR SpMV calls of the "
                                                   f"oracle's pthreads port on all {threads} host threads (the "
                                                   "reference itself has no threading)"}
    return out


def run_spmv_dist(args, rank, world, local):
    """Row-partitioned SpMV (halo exchange over NCCL + local K1), weak
    scaling: each rank owns a config-2-sized slab."""
    import torch
    import torch.distributed as dist

    from paper_1501_00324_b200 import capi

    hbm, peak_src = peaks()
    d, ng, ro, ci, v, info = dist_operator(args, rank, world)
    nloc, nnz = ro.size - 1, int(ro[-1])
    x = torch.tensor(np.random.default_rng(1 + rank).uniform(0.1, 1.0, nloc), device="cuda")
    y = torch.empty(nloc, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        d.spmv(x, y, stream=stream)
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    l0 = capi.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            d.spmv(x, y, stream=stream)
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = capi.launch_count() - l0
    barrier(world)
    ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps, world)
    eff, alg, nnz_all = sum_over_ranks([20.0 * nnz, 12.0 * nnz + 16.0 * nloc, float(nnz)], world)
    value = eff / (ms * 1e-3) / 1e9
    per_gpu_alg = alg / world / (ms * 1e-3) / 1e9
    # end to end: host x slice in, host y slice out on every rank
    xh = x.cpu().numpy()
    k_e2e = max(3, min(args.steps, 30))
    d.spmv(xh)
    barrier(world)
    t = time.perf_counter()
    for _ in range(k_e2e):
        d.spmv(xh)
    e2e_ms = max_over_ranks((time.perf_counter() - t) * 1e3 / k_e2e, world)
    return {
        "e2e": {"value": round(eff / (e2e_ms * 1e-3) / 1e9, 2), "unit": "GB/s", "h2d_bytes_per_step": 8 * nloc,
                "d2h_bytes_per_step": 8 * nloc, "ms_per_step": round(e2e_ms, 4),
                "path": "ew_dist_spmv(EW_MEM_HOST) per rank"},
        "metric": "SpMV effective GB/s (20 B/nnz, PAPER.md:553)", "value": round(value, 2), "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 5),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded structured tet mesh, P1 elasticity element matrices)",
        "config": {"workload": f"row-partitioned fp64 SpMV, elasticity box slab of 87 node layers per GPU "
                               f"({nloc} rows/GPU)", "config": "c2-per-gpu", "kernel": "k1",
                   "partition": "z-slab row blocks; interior rows overlap the halo exchange, boundary rows after",
                   "transport": getattr(args, "transport_used", args.transport),
                   "nnz_total": int(nnz_all), "ghosts_rank0": info["nghost"],
                   "l2": "inputs larger than L2 on every GPU"},
        "roofline": {"bound": "hbm", "achieved": round(per_gpu_alg, 1), "peak": hbm, "peak_source": peak_src,
                     "unit": "GB/s", "frac": round(per_gpu_alg / hbm, 4), "traffic": None,
                     "note": "per-GPU algorithmic bytes / max-over-ranks step time (pack + exchange + SpMV)"},
        "gpu_launches": int(launches), "clocks": clk.summary(),
    }


def reference_cg_sample(ro, ci, v, rows, iters):
    """The reference's cg_solve(csr_ref) on the principal submatrix of the
    leading `rows` rows (SPD like the whole operator), b = A 1, 1 thread.
    Returns (it/s, nnz of the sample, seconds)."""
    from oracle.oracle import Csr, Reference

    F = Reference()
    end = int(ro[rows])
    keep = ci[:end] < rows
    row_of = np.repeat(np.arange(rows), np.diff(ro[:rows + 1]))
    sro = np.zeros(rows + 1, np.int64)
    np.cumsum(np.bincount(row_of[keep], minlength=rows), out=sro[1:])
    m = Csr.make(rows, rows, sro, ci[:end][keep], v[:end][keep])
    b = F.spmv_csr(m, np.ones(rows))
    t = time.perf_counter()
    res = F.cg("csr_ref", m, b, tol=1e-300, max_iterations=iters)
    dt = time.perf_counter() - t
    return res.iterations / dt, m.nnz, dt


def run_cg_dist(args, rank, world, local, shape="c2-slab"):
    """Row-partitioned Jacobi PCG, 1000 iterations per step. shape "c5":
    config 5 (100M rows) split over the ranks (strong scaling); "c2-slab":
    a config-2-sized slab per rank (weak scaling)."""
    import torch

    from paper_1501_00324_b200 import capi

    hbm, peak_src = peaks()
    d, ng, ro, ci, v, info = dist_operator(args, rank, world, shape)
    nloc, nnz = ro.size - 1, int(ro[-1])
    ones = torch.ones(d.owned, dtype=torch.float64, device="cuda")
    b = d.spmv(ones)  # b = A * 1 (ellwarp_cli.cpp:192-195)
    # diagonal of the owned rows (global column == global row)
    diag = np.zeros(nloc)
    r0 = int(info["row_begin"])
    for a in range(0, nloc, 1 << 22):  # in row chunks: config 5 at N=1 has 4.5G entries
        e = min(nloc, a + (1 << 22))
        lo, hi = int(ro[a]), int(ro[e])
        rows = np.repeat(np.arange(a, e), np.diff(ro[a:e + 1]))
        hit = ci[lo:hi] == rows + r0
        diag[rows[hit]] = v[lo:hi][hit]
    dd = torch.tensor(diag, device="cuda")
    iters = args.iterations
    # full-length warm-up steps (clocks ramp up from idle), each result held
    # while the next solve allocates its own, as in the timed loop (else the
    # allocator's second solution buffer is first allocated inside it)
    res = None
    for _ in range(args.warmup):
        res = d.cg_solve(b, dd, tol=1e-300, max_iterations=iters)
    torch.cuda.synchronize()
    barrier(world)
    l0 = capi.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ran = []
    with ClockSampler(local) as clk:
        ev0.record()
        marks = []
        for _ in range(args.steps):
            res = d.cg_solve(b, dd, tol=1e-300, max_iterations=iters)
            ran.append(res.iterations)
            marks.append(torch.cuda.Event(enable_timing=True))
            marks[-1].record()
        ev1.record()
        torch.cuda.synchronize()
    assert all(r == iters for r in ran), f"a timed solve stopped early: {ran}"
    step_ms = [round(t, 3) for t in step_times(ev0, marks)]
    launches = capi.launch_count() - l0
    ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps, world)
    it_s = sum(ran) / args.steps / (ms * 1e-3)
    nnz_all, n_all = sum_over_ranks([float(nnz), float(nloc)], world)
    b_it = 12 * nnz_all + 104 * n_all + (12 * nnz_all + 24 * n_all) / 50
    per_gpu = b_it / world * it_s / 1e9
    # the same with the bytes the partition's layouts stream (padding, grouped columns)
    (sb_all,) = sum_over_ranks([float(sum(d.info(i)["stream_bytes"] for i in range(1)))], world)
    s_it = sb_all + 104 * n_all + (sb_all + 24 * n_all) / 50
    # end to end: host b / diag in, solution + history out, every rank
    bh, dh = b.cpu().numpy(), diag
    barrier(world)
    t = time.perf_counter()
    d.cg_solve(bh, dh, tol=1e-300, max_iterations=iters)
    e2e_s = max_over_ranks(time.perf_counter() - t, world)
    strong = shape == "c5"
    if strong:
        workload = (f"row-partitioned Jacobi PCG {iters} it, config 5: 3-DOF elasticity box(321,321,321) "
                    f"= {int(n_all):,} rows, {int(nnz_all):,} nnz over {world} GPU(s), z-slab row blocks "
                    f"(rank 0: {nloc} rows)")
    else:
        workload = (f"row-partitioned Jacobi PCG {iters} it, elasticity box slab of 87 node layers per "
                    f"GPU ({nloc} rows/GPU, natural ordering)")
    out = {
        "e2e": {"value": round(iters / e2e_s, 2), "unit": "it/s", "h2d_bytes_per_step": 16 * nloc,
                "d2h_bytes_per_step": 8 * nloc + 8 * (iters + 1),
                "path": "ew_dist_cg_solve(EW_MEM_HOST) per rank: b, diag in, solution + history out"},
        "metric": "CG iterations/s", "value": round(it_s, 2), "unit": "it/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
        "scaling": "strong" if strong else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload, "config": "c5" if strong else "c5-weak",
                   "iterations_per_step": iters, "iterations_run": ran, "nrows_total": int(n_all),
                   "nnz_total": int(nnz_all), "transport": getattr(args, "transport_used", args.transport),
                   "ghosts_rank0": info["nghost"], "final_residual": float(res.residual_history[-1]),
                   "step_ms_rank0": step_ms},
        "roofline": {"bound": "hbm", "achieved": round(per_gpu, 1), "peak": hbm, "peak_source": peak_src,
                     "unit": "GB/s", "frac": round(per_gpu / hbm, 4),
                     "streamed_frac": round(s_it / world * it_s / 1e9 / hbm, 4),
                     "streamed_bytes_per_iteration": s_it,
                     "traffic": (ncu_traffic(f"c5/cg_k1_dot_strong/n{world}") if strong else ncu_traffic("c5/cg_k1_dot"))
                     if args.scale == 1.0 else None,
                     "traffic_source": "profiles/ncu_traffic.json: DRAM bytes per launch of the iteration's dominant "
                                       "kernel, the fused SpMV + p.q (one per iteration)",
                     "algorithmic_bytes_per_iteration": b_it,
                     "note": "frac: per-GPU share of 12 nnz + 104 n + refresh bytes per iteration / "
                             "max-over-ranks iteration time; streamed_frac: the same with the partition layouts' "
                             "own matrix bytes (padding, grouped columns) in place of 12 B/nnz"},
        "gpu_launches": int(launches), "clocks": clk.summary(),
    }
    if strong and rank == 0 and world == 1 and not args.no_cpu_baseline:
        rows = 3 * 322 * 322 * 8  # the first 8 node layers
        rate, snnz, dt = reference_cg_sample(ro, ci, v, rows, max(2, args.cpu_cg_iters))
        out["cpu_baseline"] = {"value": round(rate * snnz / nnz_all, 5), "unit": "it/s", "cores": 1,
                               "kind": "reference",
                               "sample": f"cg_solve(csr_ref) for {max(2, args.cpu_cg_iters)} iterations on the "
                                         f"principal submatrix of config 5's first 8 node layers ({rows} rows, "
                                         f"{snnz} nnz, {rate:.3f} it/s, {dt:.1f}s; oracle/_ref, 1 thread), "
                                         "scaled by nnz to the whole matrix"}
    return out


def cg_one_gpu(args, a, n, nc, nnz, bd, dd, b, diag, kernel, row_order, local):
    """Time `args.steps` forced-length PCG solves of one prepared kernel on
    one GPU (after `args.warmup` untimed ones). Returns the line's fields."""
    import torch

    from paper_1501_00324_b200 import capi

    hbm, peak_src = peaks()
    permuted = kernel.endswith(("r", "rs"))
    t = time.time()
    k = capi.Kernel(kernel, a, threshold=args.threshold, row_order=row_order)
    torch.cuda.synchronize()
    t_prepare = time.time() - t
    log(f"[bench] prepare({kernel}, row_order={row_order}) {t_prepare:.2f}s")
    iters = args.iterations
    res = None
    for _ in range(args.warmup):
        res = k.cg_solve(bd, dd, tol=1e-300, max_iterations=iters, permuted=permuted)
    torch.cuda.synchronize()
    l0 = capi.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ran, marks, host = [], [], []
    with ClockSampler(local) as clk:
        ev0.record()
        for _ in range(args.steps):
            th = time.perf_counter()
            res = k.cg_solve(bd, dd, tol=1e-300, max_iterations=iters, permuted=permuted)
            host.append(round((time.perf_counter() - th) * 1e3, 1))
            ran.append(res.iterations)
            marks.append(torch.cuda.Event(enable_timing=True))
            marks[-1].record()
        ev1.record()
        torch.cuda.synchronize()
    assert all(r == iters for r in ran), f"a timed solve stopped early: {ran}"
    step_ms = [round(t, 3) for t in step_times(ev0, marks)]
    launches = capi.launch_count() - l0
    ms = ev0.elapsed_time(ev1) / args.steps
    it_s = sum(ran) / args.steps / (ms * 1e-3)
    kinfo = k.info()
    slots, narrow = int(kinfo.stored_slots), int(kinfo.narrow_slots)
    b_it = 12 * nnz + 104 * n + (12 * nnz + 24 * n) / 50
    # the bytes the layout streams instead of 12 B/nnz (padding; 16-bit columns)
    lay_bytes = 8 * slots + int(kinfo.col_stream_bytes)
    s_it = b_it + (lay_bytes - 12 * nnz) * (1 + 1 / 50)
    # dominant kernel: the SpMV (~2/3 of an iteration), timed alone with CUDA
    # events on its stream, x (a CG direction) L2-resident as in the solve
    stream = torch.cuda.current_stream()
    xs = torch.tensor(np.random.default_rng(1).uniform(0.1, 1.0, nc), device="cuda")
    ys = torch.empty(n, dtype=torch.float64, device="cuda")
    spmv = k.apply_permuted if k.has_perm else k.apply
    for _ in range(5):
        spmv(xs, ys, stream=stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(50):
        spmv(xs, ys, stream=stream)
    e1.record(stream)
    e1.synchronize()
    t_k = e0.elapsed_time(e1) * 1e-3 / 50
    alg = 12 * nnz + 8 * n + 8 * nc
    key = f"{args.config}/cg_k1_dot/{row_order}"
    # end to end through ew_cg_solve[_permuted] with host b / diag / x
    t = time.perf_counter()
    reps = max(1, min(args.steps, 2))
    for _ in range(reps):
        r2 = k.cg_solve(b, diag, tol=1e-300, max_iterations=iters, permuted=permuted)
        assert r2.iterations == iters
    e2e_s = (time.perf_counter() - t) / reps
    return {
        "value": round(it_s, 2), "ms_per_step": round(ms, 4), "row_order": row_order,
        "iterations_run": ran, "stored_slots": slots, "prepare_s": round(t_prepare, 3),
        "step_ms": step_ms, "step_host_ms": host, "gpu_launches": int(launches), "clocks": clk.summary(),
        "roofline": {"bound": "hbm", "achieved": round(alg / t_k / 1e9, 1), "peak": hbm, "peak_source": peak_src,
                     "unit": "GB/s", "frac": round(alg / t_k / 1e9 / hbm, 4),
                     "streamed_frac": round((lay_bytes + 8 * n + 8 * nc) / t_k / 1e9 / hbm, 4),
                     "traffic": ncu_traffic(key) if args.scale == 1.0 else None,
                     "traffic_source": f"profiles/ncu_traffic.json[{key}] (the CG's SpMV+p.q kernel)",
                     "kernel": "k1_kernel (apply_permuted)" if k.has_perm else "k1_kernel",
                     "kernel_us": round(t_k * 1e6, 2), "algorithmic_bytes_per_launch": alg},
        "iteration_roofline": {"bound": "hbm", "achieved": round(b_it * it_s / 1e9, 1), "peak": hbm,
                               "unit": "GB/s", "frac": round(b_it * it_s / 1e9 / hbm, 4),
                               "streamed_frac": round(s_it * it_s / 1e9 / hbm, 4),
                               "algorithmic_bytes_per_iteration": b_it, "streamed_bytes_per_iteration": s_it,
                               "note": "frac: 12 nnz + 104 n + refresh share per iteration / iteration time; "
                                       "streamed_frac: the same with the layout's own matrix bytes (padding, "
                                       "16-bit columns) in place of 12 B/nnz"},
        "e2e": {"value": round(iters / e2e_s, 2), "unit": "it/s", "h2d_bytes_per_step": 16 * n,
                "d2h_bytes_per_step": 8 * n + 8 * (iters + 1),
                "path": "ew_cg_solve_permuted(EW_MEM_HOST): b, diag in, solution + history out"},
    }


def run_cg(args, rank, world, local):
    """Jacobi PCG on one GPU (config 4 by default): the kernel in the row
    order(s) asked for, 1000 forced iterations per step."""
    if world > 1 or args.config == "c5":
        return run_cg_dist(args, rank, world, local, shape="c5")
    import torch

    from paper_1501_00324_b200 import capi

    n, nc, ro, ci, v = build_matrix(args.config, args.scale)
    nnz = int(ro[-1])
    a = capi.Csr(n, nc, ro, ci, v)
    diag = a.extract_diagonal()
    b = a.spmv(np.ones(nc))  # b = A * 1 (ellwarp_cli.cpp:192-195)
    bd = torch.tensor(b, device="cuda")
    dd = torch.tensor(diag, device="cuda")
    orders = [args.row_order]
    if args.kernel.endswith(("r", "rs")) and args.both_orders:
        orders = ["locality", "reference"] if args.row_order == "locality" else ["reference", "locality"]
    lines = []
    for order in orders:
        lines.append(cg_one_gpu(args, a, n, nc, nnz, bd, dd, b, diag, args.kernel, order, local))
        torch.cuda.empty_cache()
    del a
    first = lines[0]
    out = {
        "metric": "CG iterations/s", "value": first["value"], "unit": "it/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": first["ms_per_step"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": CONFIGS[args.config]["name"], "config": args.config, "kernel": args.kernel,
                   "row_order": first["row_order"], "iterations_per_step": args.iterations, "nrows": n,
                   "nnz": nnz, "stored_slots": first["stored_slots"], "prepare_s": first["prepare_s"],
                   "iterations_run": first["iterations_run"], "step_ms_rank0": first["step_ms"],
                   "step_host_ms_rank0": first["step_host_ms"]},
        "roofline": first["roofline"], "iteration_roofline": first["iteration_roofline"], "e2e": first["e2e"],
        "gpu_launches": first["gpu_launches"], "clocks": first["clocks"],
    }
    for other in lines[1:]:
        out[f"{other['row_order']}_row_order"] = {kk: other[kk] for kk in (
            "value", "ms_per_step", "iterations_run", "stored_slots", "prepare_s", "step_ms", "roofline",
            "iteration_roofline", "e2e", "gpu_launches", "clocks")}
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.config != "c5full":
        rate, its, dt = reference_cg_rate(n, nc, ro, ci, v, iters=max(2, args.cpu_cg_iters))
        out["cpu_baseline"] = {"value": round(rate, 3), "unit": "it/s", "cores": 1, "kind": "reference",
                               "sample": f"cg_solve(csr_ref) {its} iterations on the full matrix "
                                         f"({dt:.1f}s, oracle/_ref, 1 thread)"}
    return out


# Config 3: the paper's 15-matrix suite (Table 2) at its
# Table 2 sizes: seeded stand-ins whose nz / nrows / minrow / maxrow are
# Table 2's (workloads.TABLE2, table2_matrix; tests/test_workloads.py).
def suite_names():
    from paper_1501_00324_b200 import workloads as W

    return [t[0] for t in W.TABLE2]


def run_suite(args):
    """Config 3: every kernel id on the 15 structures, L2 flushed before each
    timed launch (the paper's "1 iteration" protocol)."""
    import torch

    from paper_1501_00324_b200 import capi, load_ellwarp

    ew_mod = load_ellwarp()
    torch.cuda.set_device(0)
    hbm, peak_src = peaks()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MB > L2
    # k1rs_loc / k2rs_loc: the r/rs kernels in the locality row order (extension)
    kernels = ["k1", "k1rs", "k2", "csr_ref", "csr_vector", "ell", "hyb", "coo", "k1rs_loc", "k2rs_loc"]
    rows = []
    stream = torch.cuda.current_stream()
    from paper_1501_00324_b200 import workloads as W

    table = {t[0]: t for t in W.TABLE2}
    only = set(args.suite_only.split(",")) if args.suite_only else None
    for name in suite_names():
        if only and name not in only:
            continue
        t = time.time()
        mn, mc, ro, ci, v = W.table2_matrix(name, ew_mod)
        lens = np.diff(ro)
        a = capi.Csr(mn, mc, ro, ci, v)
        nnz = a.nnz
        m = argparse.Namespace(nrows=mn, ncols=mc)
        x = torch.tensor(np.random.default_rng(1).uniform(0.1, 1.0, m.ncols), device="cuda")
        y = torch.empty(m.nrows, dtype=torch.float64, device="cuda")
        kind, spec = W.table2_spec(name)
        _, t_nnz, t_rows, t_min, t_max = table[name]
        rec = {"matrix": name, "nrows": m.nrows, "nnz": nnz, "minrow": int(lens.min()), "maxrow": int(lens.max()),
               "table2": {"nz": t_nnz, "nrows": t_rows, "minrow": t_min, "maxrow": t_max},
               "generator": {"kind": kind, **{k2: (round(v2, 6) if isinstance(v2, float) else v2)
                                              for k2, v2 in spec.items()}},
               "gen_s": round(time.time() - t, 1)}
        for kid in kernels:
            sweep = [int(t) for t in args.suite_thresholds.split(",")] if args.suite_thresholds else [4, 8, 12, 16, 20, 24, 32]
            thresholds = [0] if not kid.startswith("k2") else sorted(set(sweep) | {max(1, int(lens.max()))})
            best = None
            for th in thresholds:
                try:
                    loc = kid.endswith("_loc")
                    k = capi.Kernel(kid[:-4] if loc else kid, a, threshold=th,
                                    row_order="locality" if loc else "reference")
                except capi.DeviceError as e:  # e.g. ELL padding beyond HBM (webbase)
                    rec[kid] = f"oom: {str(e)[:60]}"
                    break
                fn = k.apply_permuted if k.has_perm else k.apply
                times, warm = [], []
                for it in range(args.suite_iters + 1):
                    # cold: K x (L2 flush by reading 256 MB, launch) minus K x flush alone
                    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
                    K = 8
                    e[0].record(stream)
                    for _ in range(K):
                        capi.l2_flush(flush, stream=stream)  # displaces the evict_last x lines too
                        fn(x, y, stream=stream)
                    e[1].record(stream)
                    for _ in range(K):
                        capi.l2_flush(flush, stream=stream)
                    e[2].record(stream)
                    for _ in range(4 * K):  # warm: back to back, L2-resident when it fits
                        fn(x, y, stream=stream)
                    e[3].record(stream)
                    e[3].synchronize()
                    if it >= 1:
                        times.append(max(1e-7, (e[0].elapsed_time(e[1]) - e[1].elapsed_time(e[2])) * 1e-3 / K))
                        warm.append(e[2].elapsed_time(e[3]) * 1e-3 / (4 * K))
                med = float(np.median(times))
                if best is None or med < best[0]:
                    best = (med, th, k.stored_slots, float(np.median(warm)))
                del k
            if best is None:
                continue
            med, th, slots, wmed = best
            rec[kid] = {"us": round(med * 1e6, 2), "eff_gbs": round(20 * nnz / med / 1e9, 1),
                        "alg_gbs": round((12 * nnz + 16 * m.nrows) / med / 1e9, 1), "stored_slots": int(slots),
                        "warm_us": round(wmed * 1e6, 2), "warm_eff_gbs": round(20 * nnz / wmed / 1e9, 1)}
            if kid.startswith("k2"):
                rec[kid]["threshold"] = int(th)
        log(f"[suite] {name}: " + ", ".join(f"{k}={rec[k]['eff_gbs'] if isinstance(rec[k], dict) else rec[k]}"
                                             for k in kernels if k in rec))
        rows.append(rec)
        del a
        torch.cuda.empty_cache()
    paper_ids = [kk for kk in kernels if not kk.endswith("_loc")]
    best_k = {r["matrix"]: max((kk for kk in paper_ids if isinstance(r.get(kk), dict)),
                               key=lambda kk: r[kk]["eff_gbs"]) for r in rows}
    best_all = {r["matrix"]: max((kk for kk in kernels if isinstance(r.get(kk), dict)),
                                 key=lambda kk: r[kk]["eff_gbs"]) for r in rows}
    return {"metric": "SpMV effective GB/s per matrix (20 B/nnz), L2 flushed (evict_last read of 256 MB) before each launch; "
                      "warm_*: back-to-back launches",
            "workload": "config 3: 15 seeded stand-ins with Table 2's nz / nrows / minrow / maxrow "
                        "(workloads.TABLE2; generator kinds of bench/fetch.cpp)",
            "unit": "GB/s", "peak": hbm, "peak_source": peak_src, "iterations": args.suite_iters,
            "fastest_kernel": best_k,
            "fastest_including_locality_order": best_all,
            "k1_or_k2_fastest": sum(1 for v in best_k.values() if v.startswith("k")),
            "rows": rows}


def run_alpha(args):
    """the paper's break-even analysis (Table 5,
    PAPER.md:598-626; analyze_alpha, bench.cpp:252-319) on the device.
    t_base: baseline SpMV; t_kernel: reordered kernel in permuted space;
    t_reorder: bulk_scatter = values-only refresh through the slot map,
    host_loop = full device rebuild (sort + renumber + layout).
    alpha = compute_alpha(t_reorder, t_kernel, t_base)."""
    import torch

    from paper_1501_00324_b200 import capi, load_ellwarp

    ew_mod = load_ellwarp()
    torch.cuda.set_device(0)
    stream = torch.cuda.current_stream()

    def time_dev(fn, reps):
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e-3)
        return float(np.median(ts))

    def time_host(fn, reps):
        ts = []
        for _ in range(reps):
            torch.cuda.synchronize()
            t = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t)
        return float(np.median(ts))

    from paper_1501_00324_b200 import workloads as W

    rows = []
    for name in suite_names():
        mn, mc, ro, ci, v = W.table2_matrix(name, ew_mod)
        a = capi.Csr(mn, mc, ro, ci, v)
        m = argparse.Namespace(nrows=mn, ncols=mc)
        x = torch.tensor(np.random.default_rng(1).uniform(0.1, 1.0, m.ncols), device="cuda")
        y = torch.empty(m.nrows, dtype=torch.float64, device="cuda")
        base = capi.Kernel("csr_ref", a)
        t_base = time_dev(lambda: base.apply(x, y, stream=stream), args.alpha_reps)
        for kid in ("k1rs", "k2rs"):
            k = capi.Kernel(kid, a)
            t_kernel = time_dev(lambda: k.apply_permuted(x, y, stream=stream), args.alpha_reps)
            t_bulk = time_dev(lambda: k.refresh_values(a, stream=stream), args.alpha_reps)
            t_rebuild = time_host(lambda: capi.Kernel(kid, a), max(3, args.alpha_reps // 3))
            rows.append({"matrix": name, "nnz": a.nnz, "kernel": kid, "baseline": "csr_ref",
                         "t_base_us": round(t_base * 1e6, 2), "t_kernel_us": round(t_kernel * 1e6, 2),
                         "t_reorder_bulk_us": round(t_bulk * 1e6, 2), "t_reorder_rebuild_us": round(t_rebuild * 1e6, 1),
                         "alpha_bulk": capi.compute_alpha(t_bulk, t_kernel, t_base),
                         "alpha_rebuild": capi.compute_alpha(t_rebuild, t_kernel, t_base)})
            log(f"[alpha] {name} {kid}: base {t_base*1e6:.1f}us kernel {t_kernel*1e6:.1f}us "
                f"bulk {t_bulk*1e6:.1f}us rebuild {t_rebuild*1e3:.2f}ms -> alpha {rows[-1]['alpha_bulk']} / "
                f"{rows[-1]['alpha_rebuild']}")
            del k
        del a, base
        torch.cuda.empty_cache()
    return {"metric": "alpha: SpMV calls to amortise the reorder (None = never)", "workload":
            "config 3 structures, reordered kernel vs csr_ref, device timings (warm)", "rows": rows}


def run_reference(args, rank, world):
    if rank != 0:
        return None
    n, nc, ro, ci, v = build_matrix(args.config, args.scale)
    nnz = int(ro[-1])
    cores = 1
    if args.workload == "cg":
        rate, its, dt = reference_cg_rate(n, nc, ro, ci, v, iters=max(2, args.cpu_cg_iters))
        return {"impl": "reference", "metric": "CG iterations/s", "value": round(rate, 3), "unit": "it/s",
                "n_gpus": world, "steps": 1, "warmup": 0, "higher_is_better": True,
                "config": {"workload": CONFIGS[args.config]["name"]},
                "cpu_baseline": {"kind": "reference", "cores": cores, "host_cores": os.cpu_count(),
                                 "value": round(rate, 3),
                                 "sample": f"{its} iterations cg_solve(csr_ref)"},
                "e2e": {"value": round(rate, 3), "unit": "it/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
    med, calls, t_prep = reference_spmv_rate(n, nc, ro, ci, v, kernel=args.kernel,
                                             budget_s=min(60.0, 3.0 * max(1, args.steps)),
                                             max_calls=max(args.steps, 1), warmup=args.warmup)
    val = 20 * nnz / med / 1e9
    return {"impl": "reference", "metric": "SpMV effective GB/s (20 B/nnz, PAPER.md:553)", "value": round(val, 3),
            "unit": "GB/s", "n_gpus": world, "steps": calls, "warmup": args.warmup, "ms_per_step": round(med * 1e3, 3),
            "higher_is_better": True, "dtype": "f64",
            "config": {"workload": CONFIGS[args.config]["name"], "config": args.config, "kernel": args.kernel},
            "cpu_baseline": {"kind": "reference", "cores": cores, "host_cores": os.cpu_count(),
                             "value": round(val, 3), "unit": "GB/s",
                             "sample": f"median of {calls} prepare_kernel('{args.kernel}').apply calls, full matrix "
                                       "(oracle/_ref compiled from the reference sources; single-threaded "
                                       "by construction)"},
            "e2e": {"value": round(val, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=None)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--workload", choices=["spmv", "cg", "suite", "alpha"], default="spmv")
    p.add_argument("--alpha-reps", type=int, default=9)
    p.add_argument("--suite-iters", type=int, default=5)
    p.add_argument("--suite-only", default="", help="comma-separated Table 2 names (suite workload)")
    p.add_argument("--suite-thresholds", default="", help="K2 thresholds to sweep (suite; default 4,8,12,16,20,24,32 + maxrow)")
    p.add_argument("--config", default=None)
    p.add_argument("--kernel", default=None)
    p.add_argument("--threshold", type=int, default=0)
    p.add_argument("--permuted", action="store_true")
    p.add_argument("--transport", choices=["ipc", "nccl"], default="ipc",
                   help="multi-GPU halo / dot transport (N > 1)")
    p.add_argument("--row-order", choices=["reference", "locality"], default=None,
                   help="r/rs kernels: reference sort_rows_desc order or the locality (Cuthill-McKee) order")
    p.add_argument("--scale", type=float, default=1.0, help="mesh edge scale (tests only)")
    p.add_argument("--iterations", type=int, default=1000)
    p.add_argument("--cpu-cg-iters", type=int, default=20)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cg-steps", type=int, default=10,
                   help="spmv workload: also time this many 1000-iteration CG steps of config 4 (N=1) and "
                        "config 5 (partitioned over the N GPUs; at most 3 steps) (0: skip)")
    p.add_argument("--both-orders", type=int, default=1,
                   help="CG on an r / rs kernel: also time the other row order (reference / locality)")
    args = p.parse_args()
    args.warmup = max(3, args.warmup)
    if args.config is None:
        args.config = "c4" if args.workload == "cg" else "c2"
    if args.kernel is None:
        args.kernel = "k1rs" if args.workload == "cg" else "k1"
    if args.workload == "cg":
        args.permuted = args.permuted or args.kernel.endswith(("r", "rs"))
    if args.steps is None:
        args.steps = 10 if args.workload == "cg" else 2000
    if args.row_order is None:
        # CG on an r / rs kernel: the locality row order (same row sums,
        # EW_ROW_ORDER_LOCALITY); everything else the reference's order
        args.row_order = "locality" if args.workload == "cg" and args.kernel.endswith(("r", "rs")) else "reference"
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        out = run_reference(args, rank, int(os.environ.get("WORLD_SIZE", "1")))
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    rank, world, local = dist_init(args.gpus)
    if args.workload in ("suite", "alpha"):
        if rank == 0:
            print(json.dumps(run_suite(args) if args.workload == "suite" else run_alpha(args)), flush=True)
        return
    out = run_spmv(args, rank, world, local) if args.workload == "spmv" else run_cg(args, rank, world, local)
    if args.workload == "spmv" and args.cg_steps > 0:
        # BASELINE.json's second metric beside the headline: CG iterations/s
        # on config 4 (one GPU, N=1 only) and on config 5 partitioned over
        # the N GPUs (the same 100M-row mesh at every N: strong scaling)
        import gc

        import torch

        keys = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "scaling", "config",
                "roofline", "iteration_roofline", "e2e", "gpu_launches", "clocks", "cpu_baseline",
                "reference_row_order")
        if world == 1:
            gc.collect()
            torch.cuda.empty_cache()
            c4 = argparse.Namespace(**vars(args))
            c4.steps, c4.workload, c4.config, c4.kernel = args.cg_steps, "cg", "c4", "k1rs"
            c4.permuted, c4.row_order, c4.warmup = True, "locality", 3
            line = run_cg(c4, rank, world, local)
            out["cg_c4"] = {kk: line[kk] for kk in keys if kk in line}
        gc.collect()
        torch.cuda.empty_cache()
        c5 = argparse.Namespace(**vars(args))
        c5.steps, c5.workload, c5.warmup = min(3, args.cg_steps), "cg", 1
        cg = run_cg_dist(c5, rank, world, local, shape="c5")
        if rank == 0:
            out["cg"] = {kk: cg[kk] for kk in keys if kk in cg}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Shared expectations for the GPU parity tests: what the reference computes
for prepare_kernel(id).apply / apply_permuted (kernels.cpp:23-125), restated
with the C oracle."""
import contextlib

import numpy as np


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.int64)


def default_threshold(m, t):
    # kernels.cpp:16-21
    if t > 0:
        return t
    return max(1, int(np.diff(m.row_offsets).max()) if m.nrows else 1)


def oracle_apply(R, kid, m, x, warp_size=32, threshold=0, permuted=False):
    """prepare_kernel(kid).apply(x) (or apply_permuted) restated."""
    x = np.asarray(x, np.float64)
    if kid == "csr_ref":
        return R.spmv_csr(m, x)
    k2 = kid.startswith("k2")
    t = default_threshold(m, threshold)
    op = m
    if len(kid) > 2:
        op, _ = R.reorder(m, kid.endswith("rs"))
    lay = R.build_k2(op, t, warp_size=warp_size) if k2 else R.build_k1(op, warp_size=warp_size)
    try:
        if len(kid) == 2:
            return R.spmv_layout(lay, x, scatter=True)
        if permuted:
            return R.spmv_layout(lay, x, scatter=False)
        return R.spmv_layout(lay, x[lay.forward], scatter=True)
    finally:
        R.free(lay)


def rel_close(a, b, tol):
    """almost_equal per entry (types.hpp:21-25): pure relative, exact zero equal."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    eq = a == b
    scale = np.maximum(np.abs(a), np.abs(b))
    return bool(np.all(eq | (np.abs(a - b) <= tol * scale)))


def same(a, b):
    """Bitwise equal, except that any two NaNs match (payloads differ between
    the x86 and sm_100a NaN canonicalisation)."""
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    if a.shape != b.shape:
        return False
    na, nb = np.isnan(a), np.isnan(b)
    return bool(np.array_equal(na, nb) and np.array_equal(bits(a[~na]), bits(b[~nb])))


@contextlib.contextmanager
def mps_environment(tmpdir):
    """A private CUDA MPS control daemon (pipe and log directories under
    tmpdir) for test processes that must run CONCURRENTLY on one GPU: without
    MPS, processes time-slice the GPU, and the peer transport's spin waits
    (one rank's kernel waiting on another rank's store) then depend on the
    slicing. Yields the environment for the child processes, or None when
    MPS is unavailable (the callers then fall back to time-slicing). On one
    GPU per process, the deployment layout, none of this applies."""
    import os
    import shutil
    import subprocess

    exe = shutil.which("nvidia-cuda-mps-control")
    if not exe:
        yield None
        return
    pipe, log = os.path.join(str(tmpdir), "mps_pipe"), os.path.join(str(tmpdir), "mps_log")
    os.makedirs(pipe, exist_ok=True)
    os.makedirs(log, exist_ok=True)
    env = dict(os.environ, CUDA_MPS_PIPE_DIRECTORY=pipe, CUDA_MPS_LOG_DIRECTORY=log)
    try:
        started = subprocess.run([exe, "-d"], env=env, timeout=30, capture_output=True).returncode == 0
    except (OSError, subprocess.SubprocessError):
        started = False
    if not started:
        yield None
        return
    try:
        yield env
    finally:
        try:
            subprocess.run([exe], input="quit\n", text=True, env=env, timeout=60, capture_output=True)
        except (OSError, subprocess.SubprocessError):
            pass

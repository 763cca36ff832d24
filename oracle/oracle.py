"""ctypes front-end for the two CPU oracles. TEST INFRASTRUCTURE ONLY.

* ``Restatement`` -> oracle/lib/libew_oracle.so, the C restatement
  (oracle/ew_oracle.c) of the reference hot path.
* ``Reference``   -> oracle/_ref/libellwarp_ref.so, the reference's own sources
  compiled by oracle/Makefile (present wherever ``make -C oracle`` ran in
  the container that holds /root/reference; the built .so travels to the GPU
  box with the snapshot).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs import this module. The product package
(paper_1501_00324_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATEMENT_SO = os.path.join(HERE, "lib", "libew_oracle.so")
REFERENCE_SO = os.path.join(HERE, "_ref", "libellwarp_ref.so")

_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)


def _ip(a):
    return a.ctypes.data_as(_i64p)


def _fp(a):
    return a.ctypes.data_as(_f64p)


@dataclass
class Csr:
    """Host CSR with the reference's int64/double types (csr.hpp:26-36)."""

    nrows: int
    ncols: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray

    @property
    def nnz(self):
        return int(self.col_indices.size)

    @staticmethod
    def make(nrows, ncols, ro, ci, v):
        return Csr(int(nrows), int(ncols), np.ascontiguousarray(ro, np.int64),
                   np.ascontiguousarray(ci, np.int64), np.ascontiguousarray(v, np.float64))

    def args(self):
        return (C.c_int64(self.nrows), C.c_int64(self.ncols), _ip(self.row_offsets),
                _ip(self.col_indices), _fp(self.values))


class OracleError(Exception):
    def __init__(self, code, msg=""):
        super().__init__(msg or f"oracle status {code}")
        self.code = code


# ----------------------------------------------------------------------------
# C restatement
# ----------------------------------------------------------------------------
class _Layout(C.Structure):
    _fields_ = [("kind", C.c_int), ("warp_size", C.c_int64), ("nrows", C.c_int64),
                ("ncols", C.c_int64), ("nnz", C.c_int64), ("threshold", C.c_int64),
                ("nwarps", C.c_int64), ("nslots", C.c_int64), ("row_major", C.c_int),
                ("values", _f64p), ("col_indices", _i64p), ("warp_offset", _i64p),
                ("maxrows", _i64p), ("rows_in_warp", _i64p), ("reduction", _i64p),
                ("rows_offset_warp", _i64p), ("forward", _i64p), ("inverse", _i64p),
                ("sorted_row_length", _i64p)]


class _CgCfg(C.Structure):
    _fields_ = [("rel_tolerance", C.c_double), ("max_iterations", C.c_int64),
                ("jacobi", C.c_int), ("recompute_interval", C.c_int64),
                ("divergence_limit", C.c_double)]


class _CgRes(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("converged", C.c_int), ("spmv_calls", C.c_int64),
                ("history_len", C.c_int64)]


@dataclass
class Layout:
    """numpy view of a WarpLayoutK1/K2 (warp_layout.hpp:13-61)."""

    kind: str
    warp_size: int
    nrows: int
    ncols: int
    nnz: int
    threshold: int
    values: np.ndarray
    col_indices: np.ndarray
    warp_offset: np.ndarray
    maxrows: np.ndarray
    rows_in_warp: np.ndarray
    forward: np.ndarray
    sorted_row_length: np.ndarray
    reduction: np.ndarray | None = None
    rows_offset_warp: np.ndarray | None = None
    stored_slots: int = 0
    _ptr: object = None

    @property
    def nwarps(self):
        return int(self.warp_offset.size)

    @property
    def padded_slots(self):
        return self.stored_slots - self.nnz


@dataclass
class CgResult:
    solution: np.ndarray
    iterations: int
    residual_history: np.ndarray
    converged: bool
    spmv_calls: int


def _cg_cfg(tol, max_it, jacobi, recompute, divergence):
    return _CgCfg(float(tol), int(max_it), 1 if jacobi else 0, int(recompute), float(divergence))


class Restatement:
    def __init__(self, path=RESTATEMENT_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle restatement`")
        L = self.lib = C.CDLL(path)
        L.ewo_compute_k2_lanes.restype = C.c_int64
        L.ewo_layout_stored_slots.restype = C.c_int64
        L.ewo_build_k1.argtypes = [C.c_int64, C.c_int64, _i64p, _i64p, _f64p, C.c_int, C.c_int,
                                   C.c_int, C.c_int, C.c_int, C.POINTER(C.POINTER(_Layout))]
        L.ewo_build_k2.argtypes = [C.c_int64, C.c_int64, _i64p, _i64p, _f64p, C.c_int, C.c_int,
                                   C.c_int, C.c_int64, C.c_int, C.POINTER(C.POINTER(_Layout))]
        L.ewo_layout_stored_slots.argtypes = [C.POINTER(_Layout)]
        L.ewo_spmv_layout.argtypes = [C.POINTER(_Layout), _f64p, C.c_int, _f64p]
        L.ewo_value_slot_map.argtypes = [C.POINTER(_Layout), _i64p, _i64p]
        L.ewo_cg_layout.argtypes = [C.POINTER(_Layout), C.c_int, C.c_int64, _f64p, _f64p,
                                    C.POINTER(_CgCfg), _f64p, _f64p, C.POINTER(_CgRes)]
        L.ewo_cg_layout_mt.argtypes = L.ewo_cg_layout.argtypes + [C.c_int]
        L.ewo_spmv_layout_mt.argtypes = [C.POINTER(_Layout), _f64p, C.c_int, _f64p, C.c_int]
        L.ewo_cg_solve.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, _f64p, _f64p,
                                   C.POINTER(_CgCfg), _f64p, _f64p, C.POINTER(_CgRes)]
        L.ewo_compute_k2_lanes.argtypes = [C.c_int64, C.c_int64, C.c_int64]
        csr = [C.c_int64, C.c_int64, _i64p, _i64p, _f64p]
        L.ewo_spmv_csr.argtypes = csr + [_f64p, _f64p]
        L.ewo_extract_diagonal.argtypes = csr + [_f64p]
        L.ewo_validate_csr.argtypes = [C.c_int64, C.c_int64, C.c_int64, _i64p, C.c_int64, _i64p]
        L.ewo_sort_rows_desc.argtypes = [C.c_int64, _i64p, _i64p, _i64p]
        L.ewo_reorder.argtypes = csr + [_i64p, _i64p, C.c_int, _i64p, _f64p]
        L.ewo_layout_free.argtypes = [C.POINTER(_Layout)]
        L.ewo_compute_alpha.argtypes = [C.c_double, C.c_double, C.c_double, _i64p, C.POINTER(C.c_int)]
        self._csr_op = C.cast(L.ewo_csr_op, C.c_void_p)

    # csr.cpp
    def spmv_csr(self, m: Csr, x):
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty(m.nrows, np.float64)
        self.lib.ewo_spmv_csr(C.c_int64(m.nrows), C.c_int64(m.ncols), _ip(m.row_offsets),
                              _ip(m.col_indices), _fp(m.values), _fp(x), _fp(y))
        return y

    def spmv_csr_mt(self, m: Csr, x, threads, y=None):
        """Row-parallel pthreads port (bench CPU comparison only)."""
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty(m.nrows, np.float64) if y is None else y
        self.lib.ewo_spmv_csr_mt(C.c_int64(m.nrows), C.c_int64(m.ncols), _ip(m.row_offsets),
                                 _ip(m.col_indices), _fp(m.values), _fp(x), _fp(y), C.c_int(int(threads)))
        return y

    def extract_diagonal(self, m: Csr):
        d = np.empty(m.nrows, np.float64)
        self.lib.ewo_extract_diagonal(C.c_int64(m.nrows), C.c_int64(m.ncols), _ip(m.row_offsets),
                                      _ip(m.col_indices), _fp(m.values), _fp(d))
        return d

    def validate_csr(self, nrows, ncols, ro, ci):
        ro = np.ascontiguousarray(ro, np.int64)
        ci = np.ascontiguousarray(ci, np.int64)
        if ro.size == 0:
            return False
        return self.lib.ewo_validate_csr(C.c_int64(nrows), C.c_int64(ncols), C.c_int64(ro.size),
                                         _ip(ro), C.c_int64(ci.size), _ip(ci)) == 0

    def sort_rows_desc(self, m: Csr):
        fwd = np.empty(m.nrows, np.int64)
        inv = np.empty(m.nrows, np.int64)
        self.lib.ewo_sort_rows_desc(C.c_int64(m.nrows), _ip(m.row_offsets), _ip(fwd), _ip(inv))
        return fwd, inv

    def compute_k2_lanes(self, nnz_row, threshold, warp_size=32):
        r = self.lib.ewo_compute_k2_lanes(nnz_row, threshold, warp_size)
        if r < 0:
            raise OracleError(1, "compute_k2_lanes: invalid argument")
        return int(r)

    def _wrap(self, p):
        s = p.contents
        nw, ns, n = s.nwarps, s.nslots, s.nrows

        def arr(ptr, k, dt):
            if not ptr:
                return None
            return np.ctypeslib.as_array(ptr, shape=(max(k, 1),))[:k].astype(dt, copy=True)

        lay = Layout(kind="k1" if s.kind == 1 else "k2", warp_size=int(s.warp_size), nrows=n,
                     ncols=s.ncols, nnz=s.nnz, threshold=s.threshold,
                     values=arr(s.values, ns, np.float64), col_indices=arr(s.col_indices, ns, np.int64),
                     warp_offset=arr(s.warp_offset, nw, np.int64), maxrows=arr(s.maxrows, nw, np.int64),
                     rows_in_warp=arr(s.rows_in_warp, nw, np.int64),
                     forward=arr(s.forward, n, np.int64),
                     sorted_row_length=arr(s.sorted_row_length, n, np.int64),
                     reduction=arr(s.reduction, nw, np.int64),
                     rows_offset_warp=arr(s.rows_offset_warp, nw, np.int64),
                     stored_slots=int(self.lib.ewo_layout_stored_slots(p)), _ptr=p)
        return lay

    def build_k1(self, m: Csr, warp_size=32, segment_bytes=128, align=True, sort_rows=True,
                 row_major=False):
        p = C.POINTER(_Layout)()
        st = self.lib.ewo_build_k1(*m.args(), warp_size, segment_bytes, int(align), int(sort_rows),
                                   int(row_major), C.byref(p))
        if st:
            raise OracleError(st, "build_k1: invalid argument")
        return self._wrap(p)

    def build_k2(self, m: Csr, threshold, warp_size=32, segment_bytes=128, align=True,
                 sort_rows=True):
        p = C.POINTER(_Layout)()
        st = self.lib.ewo_build_k2(*m.args(), warp_size, segment_bytes, int(align), int(threshold),
                                   int(sort_rows), C.byref(p))
        if st:
            raise OracleError(st, "build_k2: invalid argument")
        return self._wrap(p)

    def free(self, lay: Layout):
        if lay._ptr is not None:
            self.lib.ewo_layout_free(lay._ptr)
            lay._ptr = None

    def spmv_layout(self, lay: Layout, x, scatter=True, threads=1):
        """run_k1 / run_k2; threads > 1 splits the warps over host threads
        (same per-lane sums: bitwise the single-threaded result)."""
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty(lay.nrows, np.float64)
        if threads > 1:
            self.lib.ewo_spmv_layout_mt(lay._ptr, _fp(x), int(scatter), _fp(y), int(threads))
        else:
            self.lib.ewo_spmv_layout(lay._ptr, _fp(x), int(scatter), _fp(y))
        return y

    def value_slot_map(self, lay: Layout, m: Csr):
        out = np.empty(m.nnz, np.int64)
        self.lib.ewo_value_slot_map(lay._ptr, _ip(m.row_offsets), _ip(out))
        return out

    def reorder(self, m: Csr, sort_within_rows=False):
        fwd, inv = self.sort_rows_desc(m)
        ci = np.empty(m.nnz, np.int64)
        v = np.empty(m.nnz, np.float64)
        st = self.lib.ewo_reorder(*m.args(), _ip(fwd), _ip(inv), int(sort_within_rows), _ip(ci), _fp(v))
        if st:
            raise OracleError(st, "make_reordered_r: matrix must be square")
        return Csr(m.nrows, m.ncols, m.row_offsets.copy(), ci, v), fwd

    def _cg(self, call, n, max_it):
        x = np.empty(n, np.float64)
        hist = np.empty(max_it + 2, np.float64)
        res = _CgRes()
        st = call(x, hist, res)
        if st:
            raise OracleError(st, "cg: invalid argument" if st == 1 else "cg: divergence")
        return CgResult(x, int(res.iterations), hist[: res.history_len].copy(), bool(res.converged),
                        int(res.spmv_calls))

    def cg_csr(self, m: Csr, b, tol=1e-8, max_iterations=1000, jacobi=True, recompute=50,
               divergence=1e6):
        """cg_solve with the csr_ref operator (the reference's _ellwarp.cg_solve
        with kernel='csr_ref')."""
        b = np.ascontiguousarray(b, np.float64)
        diag = self.extract_diagonal(m) if jacobi else None

        class Ctx(C.Structure):
            _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("ro", _i64p), ("ci", _i64p),
                        ("v", _f64p)]

        ctx = Ctx(m.nrows, m.ncols, _ip(m.row_offsets), _ip(m.col_indices), _fp(m.values))
        cfg = _cg_cfg(tol, max_iterations, jacobi, recompute, divergence)
        return self._cg(lambda x, h, r: self.lib.ewo_cg_solve(
            self._csr_op, C.byref(ctx), m.nrows, _fp(b), _fp(diag) if diag is not None else None,
            C.byref(cfg), _fp(x), _fp(h), C.byref(r)), m.nrows, max_iterations)

    def cg_layout(self, lay: Layout, b, diag=None, permuted=False, tol=1e-8, max_iterations=1000,
                  jacobi=True, recompute=50, divergence=1e6, threads=1):
        """cg_solve / cg_solve_permuted over a layout operator. threads > 1:
        SpMV warps and vector updates on host threads, every dot product the
        reference's sequential sum -- bitwise the single-threaded history."""
        b = np.ascontiguousarray(b, np.float64)
        d = np.ascontiguousarray(diag, np.float64) if diag is not None else None
        cfg = _cg_cfg(tol, max_iterations, jacobi, recompute, divergence)
        return self._cg(lambda x, h, r: self.lib.ewo_cg_layout_mt(
            lay._ptr, int(permuted), lay.nrows, _fp(b), _fp(d) if d is not None else None,
            C.byref(cfg), _fp(x), _fp(h), C.byref(r), int(threads)), lay.nrows, max_iterations)

    def compute_alpha(self, tr, tk, tb):
        a = C.c_int64()
        f = C.c_int()
        st = self.lib.ewo_compute_alpha(C.c_double(tr), C.c_double(tk), C.c_double(tb),
                                        C.byref(a), C.byref(f))
        if st:
            raise OracleError(st, "compute_alpha: negative time")
        return int(a.value) if f.value else None


# ----------------------------------------------------------------------------
# The real reference (oracle/_ref)
# ----------------------------------------------------------------------------
class Reference:
    def __init__(self, path=REFERENCE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` where /root/reference exists")
        L = self.lib = C.CDLL(path)
        L.refw_last_error.restype = C.c_char_p
        L.refw_bag_str.restype = C.c_char_p
        for f in ("refw_bag_ilen", "refw_bag_dlen", "refw_bag_scalar", "refw_compute_k2_lanes"):
            getattr(L, f).restype = C.c_int64
        L.refw_powerlaw_rows.argtypes = [C.c_int64, C.c_double, C.c_int64, C.c_uint64, C.c_int64,
                                         C.c_void_p]
        L.refw_random_csr.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_uint64, C.c_double,
                                      C.c_void_p]
        L.refw_cg.argtypes = [C.c_char_p, C.c_int64, C.c_int64, _i64p, _i64p, _f64p, _f64p,
                              C.c_double, C.c_int64, C.c_int, C.c_int64, C.c_double, C.c_int,
                              C.c_int, C.c_int64, C.c_void_p]
        L.refw_compute_alpha.argtypes = [C.c_double, C.c_double, C.c_double, _i64p, C.POINTER(C.c_int)]
        L.refw_prepared_apply.argtypes = [C.c_char_p, C.c_int64, C.c_int64, _i64p, _i64p, _f64p,
                                          C.c_int, C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int,
                                          _f64p, _f64p, _i64p]
        L.refw_build_layout.argtypes = [C.c_int, C.c_int64, C.c_int64, _i64p, _i64p, _f64p,
                                        C.c_int, C.c_int, C.c_int, C.c_int64, C.c_int, C.c_int,
                                        C.c_void_p]
        L.refw_prepare.argtypes = [C.c_char_p, C.c_int64, C.c_int64, _i64p, _i64p, _f64p, C.c_int,
                                   C.c_int64, C.c_void_p]
        L.refw_prepared_run.argtypes = [C.c_void_p, C.c_int, _f64p, C.c_int64, _f64p, C.c_int64]
        L.refw_prepared_free.argtypes = [C.c_void_p]
        for f in ("refw_bag_free",):
            getattr(L, f).argtypes = [C.c_void_p]
        for f in ("refw_bag_ilen", "refw_bag_dlen", "refw_bag_scalar"):
            getattr(L, f).argtypes = [C.c_void_p, C.c_int]
        L.refw_bag_icopy.argtypes = [C.c_void_p, C.c_int, _i64p]
        L.refw_bag_dcopy.argtypes = [C.c_void_p, C.c_int, _f64p]
        L.refw_bag_str.argtypes = [C.c_void_p]
        csr = [C.c_int64, C.c_int64, _i64p, _i64p, _f64p]
        L.refw_spmv_reference.argtypes = csr + [_f64p, _f64p]
        L.refw_extract_diagonal.argtypes = csr + [_f64p]
        L.refw_sort_rows_desc.argtypes = csr + [_i64p, _i64p]
        L.refw_reorder.argtypes = csr + [C.c_int, C.c_void_p]
        L.refw_compute_k2_lanes.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.POINTER(C.c_int)]
        L.refw_generate.argtypes = [C.c_char_p, C.c_uint64, C.c_void_p]
        L.refw_laplacian3d.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_void_p]
        L.refw_fem_tet_graph.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_uint64, C.c_void_p]
        L.refw_uniform_band.argtypes = [C.c_int64, C.c_int64, C.c_void_p]
        L.refw_random_case.argtypes = [C.c_int64, C.c_void_p]
        L.refw_random_vector.argtypes = [C.c_int64, C.c_uint64, _f64p]
        L.refw_from_coo.argtypes = [C.c_int64, C.c_int64, C.c_int64, _i64p, _i64p, _f64p, C.c_void_p]
        L.refw_validate.argtypes = [C.c_int64, C.c_int64, C.c_int64, _i64p, C.c_int64, _i64p, _f64p]

    def _check(self, st):
        if st:
            raise OracleError(st, self.lib.refw_last_error().decode())

    def _bag(self, fn, *args):
        b = C.c_void_p()
        self._check(fn(*args, C.byref(b)))
        return b

    def _bi(self, b, k):
        n = self.lib.refw_bag_ilen(b, k)
        a = np.empty(max(n, 0), np.int64)
        if n > 0:
            self.lib.refw_bag_icopy(b, k, _ip(a))
        return a

    def _bd(self, b, k):
        n = self.lib.refw_bag_dlen(b, k)
        a = np.empty(max(n, 0), np.float64)
        if n > 0:
            self.lib.refw_bag_dcopy(b, k, _fp(a))
        return a

    def _csr(self, b):
        m = Csr(int(self.lib.refw_bag_scalar(b, 0)), int(self.lib.refw_bag_scalar(b, 1)),
                self._bi(b, 0), self._bi(b, 1), self._bd(b, 0))
        return m

    def _take_csr(self, fn, *args):
        b = self._bag(fn, *args)
        try:
            return self._csr(b)
        finally:
            self.lib.refw_bag_free(b)

    # generators (synth.cpp) and the reference test corpus (test_support.hpp)
    def laplacian3d(self, nx, ny, nz):
        return self._take_csr(self.lib.refw_laplacian3d, C.c_int64(nx), C.c_int64(ny), C.c_int64(nz))

    def fem_tet_graph(self, n, minrow, maxrow, seed):
        return self._take_csr(self.lib.refw_fem_tet_graph, C.c_int64(n), C.c_int64(minrow),
                              C.c_int64(maxrow), C.c_uint64(seed))

    def powerlaw_rows(self, nrows, alpha, maxrow, seed, ncols=0):
        return self._take_csr(self.lib.refw_powerlaw_rows, nrows, alpha, maxrow, seed, ncols)

    def uniform_band(self, n, row_len):
        return self._take_csr(self.lib.refw_uniform_band, C.c_int64(n), C.c_int64(row_len))

    def generate(self, spec, seed=1):
        return self._take_csr(self.lib.refw_generate, spec.encode(), C.c_uint64(seed))

    def random_case(self, i):
        return self._take_csr(self.lib.refw_random_case, C.c_int64(i))

    def random_csr(self, nrows, ncols, density, seed, empty=0.0):
        return self._take_csr(self.lib.refw_random_csr, nrows, ncols, density, seed, empty)

    def random_vector(self, n, seed):
        out = np.empty(n, np.float64)
        self.lib.refw_random_vector(C.c_int64(n), C.c_uint64(seed), _fp(out))
        return out

    def from_coo(self, nrows, ncols, rows, cols, vals):
        rows = np.ascontiguousarray(rows, np.int64)
        cols = np.ascontiguousarray(cols, np.int64)
        vals = np.ascontiguousarray(vals, np.float64)
        return self._take_csr(self.lib.refw_from_coo, C.c_int64(nrows), C.c_int64(ncols),
                              C.c_int64(rows.size), _ip(rows), _ip(cols), _fp(vals))

    # hot path
    def spmv_csr(self, m: Csr, x):
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty(m.nrows, np.float64)
        self._check(self.lib.refw_spmv_reference(*m.args(), _fp(x), _fp(y)))
        return y

    def extract_diagonal(self, m: Csr):
        d = np.empty(m.nrows, np.float64)
        self._check(self.lib.refw_extract_diagonal(*m.args(), _fp(d)))
        return d

    def sort_rows_desc(self, m: Csr):
        fwd = np.empty(m.nrows, np.int64)
        inv = np.empty(m.nrows, np.int64)
        self._check(self.lib.refw_sort_rows_desc(*m.args(), _ip(fwd), _ip(inv)))
        return fwd, inv

    def compute_k2_lanes(self, nnz_row, threshold, warp_size=32):
        st = C.c_int()
        r = self.lib.refw_compute_k2_lanes(C.c_int64(nnz_row), C.c_int64(threshold),
                                           C.c_int64(warp_size), C.byref(st))
        self._check(st.value)
        return int(r)

    def build(self, kind, m: Csr, warp_size=32, threshold=0, segment_bytes=128, align=True,
              sort_rows=True, row_major=False):
        b = self._bag(self.lib.refw_build_layout, 1 if kind == "k1" else 2, *m.args(), warp_size,
                      segment_bytes, int(align), int(threshold), int(sort_rows), int(row_major))
        try:
            lay = Layout(kind=kind, warp_size=warp_size, nrows=m.nrows, ncols=m.ncols, nnz=m.nnz,
                         threshold=threshold, values=self._bd(b, 0), col_indices=self._bi(b, 0),
                         warp_offset=self._bi(b, 1), maxrows=self._bi(b, 2),
                         rows_in_warp=self._bi(b, 3), forward=self._bi(b, 4),
                         sorted_row_length=self._bi(b, 5),
                         reduction=self._bi(b, 6) if kind == "k2" else None,
                         rows_offset_warp=self._bi(b, 7) if kind == "k2" else None,
                         stored_slots=int(self.lib.refw_bag_scalar(b, 0)))
            lay.value_slot_map = self._bi(b, 8)
            lay.dump = self.lib.refw_bag_str(b).decode()
            return lay
        finally:
            self.lib.refw_bag_free(b)

    def reorder(self, m: Csr, sort_within_rows=False):
        b = self._bag(self.lib.refw_reorder, *m.args(), int(sort_within_rows))
        try:
            return self._csr(b), self._bi(b, 2)
        finally:
            self.lib.refw_bag_free(b)

    def apply(self, kernel, m: Csr, x, warp_size=32, threshold=0, segment_bytes=128, align=True,
              hyb_k_ell=-1, permuted=False):
        """prepare_kernel(kernel).apply(x) (or apply_permuted)."""
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty(m.nrows, np.float64)
        ss = C.c_int64()
        self._check(self.lib.refw_prepared_apply(kernel.encode(), *m.args(), warp_size,
                                                 segment_bytes, int(align), threshold, hyb_k_ell,
                                                 int(permuted), _fp(x), _fp(y), C.byref(ss)))
        return y

    def prepare(self, kernel, m: Csr, warp_size=32, threshold=0):
        h = C.c_void_p()
        self._check(self.lib.refw_prepare(kernel.encode(), *m.args(), warp_size, threshold,
                                          C.byref(h)))
        return h

    def run(self, h, x, y, permuted=False):
        self._check(self.lib.refw_prepared_run(h, int(permuted), _fp(x), x.size, _fp(y), y.size))

    def free_prepared(self, h):
        self.lib.refw_prepared_free(h)

    def cg(self, kernel, m: Csr, b, tol=1e-8, max_iterations=1000, jacobi=True, recompute=50,
           divergence=1e6, permuted=False, warp_size=32, threshold=0):
        b = np.ascontiguousarray(b, np.float64)
        bag = self._bag(self.lib.refw_cg, kernel.encode(), *m.args(), _fp(b), tol, max_iterations,
                        int(jacobi), recompute, divergence, int(permuted), warp_size, threshold)
        try:
            return CgResult(self._bd(bag, 0), int(self.lib.refw_bag_scalar(bag, 0)), self._bd(bag, 1),
                            bool(self.lib.refw_bag_scalar(bag, 1)), int(self.lib.refw_bag_scalar(bag, 2)))
        finally:
            self.lib.refw_bag_free(bag)

    def compute_alpha(self, tr, tk, tb):
        a = C.c_int64()
        f = C.c_int()
        self._check(self.lib.refw_compute_alpha(tr, tk, tb, C.byref(a), C.byref(f)))
        return int(a.value) if f.value else None

    # FEM assembly (fem/mesh.cpp, fem/assembly.cpp)
    def box_elements(self, nx, ny, nz):
        self.lib.refw_box_elements.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_void_p]
        b = self._bag(self.lib.refw_box_elements, nx, ny, nz)
        try:
            return self._bi(b, 0).reshape(-1, 4), int(self.lib.refw_bag_scalar(b, 0))
        finally:
            self.lib.refw_bag_free(b)

    def box_assemble(self, nx, ny, nz, ke, re, warp_size=32):
        """assemble_spmv on box_mesh: (pattern ro, pattern ci, tangent, residual)."""
        self.lib.refw_box_assemble.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int, _f64p, _f64p, C.c_void_p]
        ke = np.ascontiguousarray(ke, np.float64)
        re = np.ascontiguousarray(re, np.float64)
        b = self._bag(self.lib.refw_box_assemble, nx, ny, nz, warp_size, _fp(ke), _fp(re))
        try:
            return self._bi(b, 0), self._bi(b, 1), self._bd(b, 0), self._bd(b, 1)
        finally:
            self.lib.refw_bag_free(b)


def reference_available():
    return os.path.exists(REFERENCE_SO)

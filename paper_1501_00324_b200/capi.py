"""ctypes binding of the C ABI in include/ellwarp_b200.h.

This is the boundary the parity tests and bench.py call through. It loads the
in-tree ``lib/libellwarp_b200.so`` and raises immediately when it is missing:
there is no CPU fallback anywhere in this package.

Status codes become the reference's exceptions (types.hpp:16-18, cg.hpp:28-30):
EW_INVALID_ARGUMENT -> ValueError (Python's std::invalid_argument, as pybind11
maps it), EW_CG_DIVERGENCE -> CgDivergenceError, EW_UNSUPPORTED ->
UnsupportedError, EW_CUDA / EW_OUT_OF_MEMORY -> DeviceError.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# EW_B200_LIB: another build of the in-tree library (A/B runs of kernel variants)
LIB_PATH = os.environ.get("EW_B200_LIB") or os.path.join(HERE, "lib", "libellwarp_b200.so")

EW_OK, EW_INVALID_ARGUMENT, EW_CG_DIVERGENCE, EW_UNSUPPORTED, EW_CUDA, EW_OUT_OF_MEMORY = range(6)
EW_MEM_HOST, EW_MEM_DEVICE = 0, 1
EW_LAYOUT_K1, EW_LAYOUT_K2 = 1, 2


class CgDivergenceError(RuntimeError):
    """ellwarp::CgDivergenceError (cg.hpp:28-30)."""


class UnsupportedError(RuntimeError):
    """Input the device path rejects (EW_UNSUPPORTED)."""


class DeviceError(RuntimeError):
    """A CUDA failure inside the library (EW_CUDA / EW_OUT_OF_MEMORY)."""


_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_vp = C.c_void_p


class WarpConfig(C.Structure):
    """WarpModelConfig (warp_model.hpp:16-25)."""

    _fields_ = [("warp_size", C.c_int32), ("block_size", C.c_int32), ("segment_bytes", C.c_int32),
                ("align_warp_offsets", C.c_int32), ("ideal_cache", C.c_int32),
                ("cache_lines", C.c_int32)]

    @staticmethod
    def make(warp_size=32, block_size=None, segment_bytes=128, align=True):
        # the reference binding's make_config: block_size = max(32, ws) (module.cpp:16-26)
        bs = block_size if block_size is not None else max(32, warp_size)
        return WarpConfig(warp_size, bs, segment_bytes, 1 if align else 0, 0, 64)


class KernelOptions(C.Structure):
    _fields_ = [("k2_threshold", C.c_int64), ("hyb_k_ell", C.c_int64), ("row_order", C.c_int64)]


ROW_ORDERS = {"reference": 0, "locality": 1}


class CgConfig(C.Structure):
    _fields_ = [("rel_tolerance", C.c_double), ("max_iterations", C.c_int64), ("jacobi", C.c_int32),
                ("recompute_interval", C.c_int64), ("divergence_limit", C.c_double)]


class CgResultC(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("converged", C.c_int32), ("spmv_calls", C.c_int64),
                ("history_len", C.c_int64)]


class LayoutInfo(C.Structure):
    _fields_ = [("kind", C.c_int32), ("warp_size", C.c_int32), ("row_major", C.c_int32),
                ("sorted", C.c_int32), ("nrows", C.c_int64), ("ncols", C.c_int64), ("nnz", C.c_int64),
                ("nwarps", C.c_int64), ("nslots", C.c_int64), ("stored_slots", C.c_int64),
                ("threshold", C.c_int64), ("device_bytes", C.c_int64), ("narrow_slots", C.c_int64),
                ("col_stream_bytes", C.c_int64)]


class LayoutArrays(C.Structure):
    _fields_ = [("values", _f64p), ("col_indices", _i64p), ("warp_offset", _i64p), ("maxrows", _i64p),
                ("rows_in_warp", _i64p), ("reduction", _i64p), ("rows_offset_warp", _i64p),
                ("forward", _i64p), ("inverse", _i64p), ("sorted_row_length", _i64p)]


class LayoutDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("warp_size", C.c_int32), ("row_major", C.c_int32),
                ("nrows", C.c_int64), ("ncols", C.c_int64), ("nnz", C.c_int64), ("nwarps", C.c_int64),
                ("nslots", C.c_int64), ("threshold", C.c_int64), ("values", _f64p),
                ("col_indices", _i64p), ("warp_offset", _i64p), ("maxrows", _i64p),
                ("rows_in_warp", _i64p), ("reduction", _i64p), ("rows_offset_warp", _i64p),
                ("forward", _i64p), ("sorted_row_length", _i64p)]


class KernelInfo(C.Structure):
    _fields_ = [("id", C.c_char * 16), ("nrows", C.c_int64), ("ncols", C.c_int64), ("nnz", C.c_int64),
                ("stored_slots", C.c_int64), ("nwarps", C.c_int64), ("has_perm", C.c_int32),
                ("layout_kind", C.c_int32), ("device_bytes", C.c_int64), ("narrow_slots", C.c_int64),
                ("col_stream_bytes", C.c_int64)]


OPERATOR_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p)

# every symbol include/ellwarp_b200.h declares, with its ctypes signature
_SIGS = {
    "ew_last_error": (C.c_char_p, []),
    "ew_status_string": (C.c_char_p, [C.c_int]),
    "ew_abi_version": (C.c_int32, []),
    "ew_kernel_id_count": (C.c_int32, []),
    "ew_kernel_id": (C.c_char_p, [C.c_int32]),
    "ew_kernel_id_supported": (C.c_int32, [C.c_char_p]),
    "ew_launch_count": (C.c_int64, []),
    "ew_l2_flush": (C.c_int, [_vp, C.c_int64, _vp]),
    "ew_csr_create": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, _vp, C.c_int64, _vp, _vp, C.c_int, C.c_int32,
                                _vp, C.POINTER(_vp)]),
    "ew_csr_destroy": (C.c_int, [_vp]),
    "ew_csr_shape": (C.c_int, [_vp, _i64p, _i64p, _i64p]),
    "ew_csr_export": (C.c_int, [_vp, _vp, _vp, _vp]),
    "ew_csr_update_values": (C.c_int, [_vp, _vp, C.c_int, _vp]),
    "ew_csr_spmv": (C.c_int, [_vp, _vp, C.c_int64, _vp, C.c_int64, C.c_int, _vp]),
    "ew_csr_extract_diagonal": (C.c_int, [_vp, _vp, C.c_int, _vp]),
    "ew_sort_rows_desc": (C.c_int, [_vp, _vp, _vp]),
    "ew_reorder": (C.c_int, [_vp, _vp, C.c_int32, C.POINTER(_vp), _vp]),
    "ew_csr_sort_rows": (C.c_int, [_vp, C.POINTER(_vp)]),
    "ew_permute": (C.c_int, [_vp, C.c_int64, _vp, _vp, C.c_int32, C.c_int, _vp]),
    "ew_compute_k2_lanes": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, _i64p]),
    "ew_layout_build": (C.c_int, [_vp, C.c_int32, C.POINTER(WarpConfig), C.c_int64, C.c_int32, C.c_int32,
                                  C.POINTER(_vp)]),
    "ew_layout_import": (C.c_int, [C.POINTER(LayoutDesc), C.POINTER(_vp)]),
    "ew_layout_destroy": (C.c_int, [_vp]),
    "ew_layout_get_info": (C.c_int, [_vp, C.POINTER(LayoutInfo)]),
    "ew_layout_export": (C.c_int, [_vp, C.POINTER(LayoutArrays)]),
    "ew_layout_value_slot_map": (C.c_int, [_vp, _vp, _vp]),
    "ew_layout_refresh_values": (C.c_int, [_vp, _vp, _vp]),
    "ew_layout_dump": (C.c_int, [_vp, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "ew_layout_spmv": (C.c_int, [_vp, _vp, C.c_int64, _vp, C.c_int64, C.c_int32, C.c_int, _vp]),
    "ew_kernel_prepare": (C.c_int, [C.c_char_p, _vp, C.POINTER(WarpConfig), C.POINTER(KernelOptions),
                                    C.POINTER(_vp)]),
    "ew_kernel_destroy": (C.c_int, [_vp]),
    "ew_kernel_get_info": (C.c_int, [_vp, C.POINTER(KernelInfo)]),
    "ew_kernel_get_perm": (C.c_int, [_vp, _vp, _vp]),
    "ew_kernel_get_layout": (C.c_int, [_vp, C.POINTER(_vp)]),
    "ew_kernel_apply": (C.c_int, [_vp, _vp, C.c_int64, _vp, C.c_int64, C.c_int, _vp]),
    "ew_kernel_apply_permuted": (C.c_int, [_vp, _vp, C.c_int64, _vp, C.c_int64, C.c_int, _vp]),
    "ew_kernel_refresh_values": (C.c_int, [_vp, _vp, _vp]),
    "ew_cg_solve": (C.c_int, [_vp, _vp, _vp, C.c_int64, C.POINTER(CgConfig), C.c_int, _vp, _vp,
                              C.POINTER(CgResultC), _vp]),
    "ew_cg_solve_permuted": (C.c_int, [_vp, _vp, _vp, C.c_int64, C.POINTER(CgConfig), C.c_int, _vp, _vp,
                                       C.POINTER(CgResultC), _vp]),
    "ew_cg_solve_operator": (C.c_int, [OPERATOR_FN, _vp, C.c_int, _vp, _vp, C.c_int64, C.POINTER(CgConfig),
                                       C.c_int, _vp, _vp, C.POINTER(CgResultC), _vp]),
    "ew_compute_alpha": (C.c_int, [C.c_double, C.c_double, C.c_double, _i64p, C.POINTER(C.c_int32)]),
    "ew_assembly_create": (C.c_int, [C.c_int64, _vp, C.c_int64, C.POINTER(WarpConfig), C.POINTER(_vp)]),
    "ew_assembly_destroy": (C.c_int, [_vp]),
    "ew_assembly_pattern": (C.c_int, [_vp, _i64p, _vp, _vp]),
    "ew_assembly_run": (C.c_int, [_vp, _vp, _vp, _vp, _vp, C.c_int, _vp]),
    "ew_assembly_run_into": (C.c_int, [_vp, _vp, _vp, _vp, _vp, C.c_int, _vp]),
    "ew_partition_rows": (C.c_int, [_vp, C.c_int64, C.c_int32, _vp]),
    "ew_nccl_unique_id": (C.c_int, [_vp]),
    "ew_dist_create": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, _vp, C.c_int64, _vp, _vp, _vp, C.c_int32,
                                 C.c_int32, C.c_int32, _vp, C.c_char_p, C.POINTER(WarpConfig),
                                 C.POINTER(KernelOptions), _vp, C.POINTER(_vp)]),
    "ew_dist_create_block": (C.c_int, [C.c_int64, C.c_int64, _vp, _vp, _vp, _vp, C.c_int32, C.c_int32, _vp,
                                       C.c_char_p, C.POINTER(WarpConfig), C.POINTER(KernelOptions), _vp,
                                       C.POINTER(_vp)]),
    "ew_dist_create_peer": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, _vp, C.c_int64, _vp, _vp, _vp, C.c_int32,
                                      C.c_char_p, C.POINTER(WarpConfig), C.POINTER(KernelOptions), _vp,
                                      C.POINTER(_vp)]),
    "ew_dist_create_block_ipc": (C.c_int, [C.c_int64, C.c_int64, _vp, _vp, _vp, _vp, C.c_int32, C.c_int32,
                                           _vp, _vp, C.c_char_p, C.POINTER(WarpConfig),
                                           C.POINTER(KernelOptions), _vp, C.POINTER(_vp)]),
    "ew_dist_plan_block": (C.c_int, [C.c_int64, _vp, _vp, _vp, C.c_int32, C.c_int32, _vp, _vp, _i64p, _vp, _vp,
                                     _vp]),
    "ew_dist_destroy": (C.c_int, [_vp]),
    "ew_dist_get_info": (C.c_int, [_vp, C.c_int32, _i64p, _i64p, _i64p, _i64p]),
    "ew_dist_get_layout_bytes": (C.c_int, [_vp, C.c_int32, _i64p, _i64p]),
    "ew_dist_spmv": (C.c_int, [_vp, _vp, _vp, C.c_int, _vp]),
    "ew_dist_cg_solve": (C.c_int, [_vp, _vp, _vp, C.POINTER(CgConfig), C.c_int, _vp, _vp, C.POINTER(CgResultC),
                                   _vp]),
    "ew_mgpu_create": (C.c_int, [C.c_int64, _vp, _vp, _vp, C.c_int32, _vp, C.c_char_p, C.POINTER(WarpConfig),
                                 C.POINTER(KernelOptions), C.POINTER(_vp)]),
    "ew_mgpu_destroy": (C.c_int, [_vp]),
    "ew_mgpu_spmv": (C.c_int, [_vp, _vp, _vp]),
    "ew_mgpu_cg_solve": (C.c_int, [_vp, _vp, _vp, C.POINTER(CgConfig), _vp, _vp, C.POINTER(CgResultC)]),
}

_lib = None


def lib():
    """The loaded C library; raises if the CUDA build is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def declared_symbols():
    return list(_SIGS)


def check(status):
    if status == EW_OK:
        return
    msg = lib().ew_last_error().decode(errors="replace")
    if status == EW_INVALID_ARGUMENT:
        raise ValueError(msg)
    if status == EW_CG_DIVERGENCE:
        raise CgDivergenceError(msg)
    if status == EW_UNSUPPORTED:
        raise UnsupportedError(msg)
    raise DeviceError(f"{msg} (status {status})")


def kernel_ids():
    L = lib()
    return [L.ew_kernel_id(i).decode() for i in range(L.ew_kernel_id_count())]


def launch_count():
    return int(lib().ew_launch_count())


def l2_flush(buf, stream=None):
    """Stream-ordered L2 flush through a device tensor (>= 2x L2) read with an
    evict_last policy (ew_l2_flush)."""
    check(lib().ew_l2_flush(_ptr(buf), buf.numel() * buf.element_size(), _stream_ptr(stream)))


# --------------------------------------------------------------------------
# buffers: numpy (host) or anything with data_ptr() (torch CUDA tensors)
# --------------------------------------------------------------------------
def _host(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _ptr(a):
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    return C.c_void_p(a.ctypes.data)


def _stream_ptr(stream):
    if stream is None:
        return None
    if hasattr(stream, "cuda_stream"):
        return C.c_void_p(stream.cuda_stream)
    return C.c_void_p(int(stream))


def _mem_of(a):
    return EW_MEM_DEVICE if hasattr(a, "data_ptr") else EW_MEM_HOST


class Csr:
    """Device-resident SparseCsr (ew_csr)."""

    def __init__(self, nrows, ncols, row_offsets, col_indices, values, stream=None, canonical=True):
        ro = row_offsets if hasattr(row_offsets, "data_ptr") else _host(row_offsets, np.int64)
        ci = col_indices if hasattr(col_indices, "data_ptr") else _host(col_indices, np.int64)
        v = values if hasattr(values, "data_ptr") else _host(values, np.float64)
        nnz = ci.numel() if hasattr(ci, "numel") else ci.size
        nv = v.numel() if hasattr(v, "numel") else v.size
        nro = ro.numel() if hasattr(ro, "numel") else ro.size
        if nv != nnz:
            raise ValueError("values/col_indices length mismatch")
        h = C.c_void_p()
        check(lib().ew_csr_create(int(nrows), int(ncols), int(nro), _ptr(ro), int(nnz), _ptr(ci), _ptr(v),
                                  _mem_of(ro), 1 if canonical else 0, _stream_ptr(stream), C.byref(h)))
        self.h = h
        self.nrows, self.ncols, self.nnz = int(nrows), int(ncols), int(nnz)

    @staticmethod
    def _wrap(h):
        obj = Csr.__new__(Csr)
        obj.h = h
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib().ew_csr_shape(h, C.byref(a), C.byref(b), C.byref(c)))
        obj.nrows, obj.ncols, obj.nnz = a.value, b.value, c.value
        return obj

    def __del__(self):
        h = getattr(self, "h", None)
        if h and _lib is not None:
            _lib.ew_csr_destroy(h)
            self.h = None

    def export(self):
        ro = np.empty(self.nrows + 1, np.int64)
        ci = np.empty(self.nnz, np.int64)
        v = np.empty(self.nnz, np.float64)
        check(lib().ew_csr_export(self.h, _ptr(ro), _ptr(ci), _ptr(v)))
        return ro, ci, v

    def update_values(self, values, stream=None):
        v = values if hasattr(values, "data_ptr") else _host(values, np.float64)
        check(lib().ew_csr_update_values(self.h, _ptr(v), _mem_of(v), _stream_ptr(stream)))

    def spmv(self, x, y=None, stream=None):
        """spmv_csr_reference on the device (bit-identical)."""
        return _apply(lambda xp, nx, yp, ny, mem, s: lib().ew_csr_spmv(self.h, xp, nx, yp, ny, mem, s),
                      x, y, self.ncols, self.nrows, stream)

    def extract_diagonal(self):
        d = np.empty(self.nrows, np.float64)
        check(lib().ew_csr_extract_diagonal(self.h, _ptr(d), EW_MEM_HOST, None))
        return d

    def sort_rows_desc(self):
        fwd = np.empty(self.nrows, np.int64)
        inv = np.empty(self.nrows, np.int64)
        check(lib().ew_sort_rows_desc(self.h, _ptr(fwd), _ptr(inv)))
        return fwd, inv

    def reorder(self, sort_within_rows=False, forward=None):
        """make_reordered_r (+ rs); forward=None renumbers by sort_rows_desc."""
        h = C.c_void_p()
        fwd = np.empty(self.nrows, np.int64)
        fin = _host(forward, np.int64) if forward is not None else None
        check(lib().ew_reorder(self.h, _ptr(fin), 1 if sort_within_rows else 0, C.byref(h), _ptr(fwd)))
        return Csr._wrap(h), (fwd if forward is None else fin.copy())

    def sort_rows(self):
        h = C.c_void_p()
        check(lib().ew_csr_sort_rows(self.h, C.byref(h)))
        return Csr._wrap(h)


def permute(forward, x, inverse=False):
    """apply_forward / apply_inverse (permutation.cpp:35-47) on the device."""
    f = _host(forward, np.int64)
    xh = _host(x, np.float64)
    if xh.size != f.size:
        raise ValueError("permutation size mismatch")
    out = np.empty(f.size, np.float64)
    check(lib().ew_permute(_ptr(f), f.size, _ptr(xh), _ptr(out), 1 if inverse else 0, EW_MEM_HOST, None))
    return out


def _apply(fn, x, y, nx, ny, stream):
    if hasattr(x, "data_ptr"):
        if y is None:
            import torch

            y = torch.empty(ny, dtype=torch.float64, device=x.device)
        check(fn(_ptr(x), nx, _ptr(y), ny, EW_MEM_DEVICE, _stream_ptr(stream)))
        return y
    xh = _host(x, np.float64)
    if xh.size != nx:
        # let the library report the reference's dimension error
        pass
    yh = np.empty(ny, np.float64) if y is None else y
    check(fn(_ptr(xh), xh.size, _ptr(yh), ny, EW_MEM_HOST, _stream_ptr(stream)))
    return yh


def compute_k2_lanes(nnz_row, threshold, warp_size=32):
    out = C.c_int64()
    check(lib().ew_compute_k2_lanes(int(nnz_row), int(threshold), int(warp_size), C.byref(out)))
    return out.value


@dataclass
class LayoutExport:
    kind: str
    warp_size: int
    nrows: int
    ncols: int
    nnz: int
    threshold: int
    stored_slots: int
    values: np.ndarray
    col_indices: np.ndarray
    warp_offset: np.ndarray
    maxrows: np.ndarray
    rows_in_warp: np.ndarray
    forward: np.ndarray
    inverse: np.ndarray
    sorted_row_length: np.ndarray
    reduction: np.ndarray | None = None
    rows_offset_warp: np.ndarray | None = None

    @property
    def nwarps(self):
        return int(self.warp_offset.size)

    @property
    def padded_slots(self):
        return self.stored_slots - self.nnz


class Layout:
    """Device WarpLayoutK1 / WarpLayoutK2 (ew_layout)."""

    def __init__(self, h, owner=None):
        self.h = h
        self._owner = owner  # a Kernel owns its layout

    @staticmethod
    def build(csr: Csr, kind="k1", warp_size=32, threshold=0, segment_bytes=128, align=True,
              sort_rows=True, row_major=False):
        cfg = WarpConfig.make(warp_size, segment_bytes=segment_bytes, align=align)
        h = C.c_void_p()
        check(lib().ew_layout_build(csr.h, EW_LAYOUT_K1 if kind == "k1" else EW_LAYOUT_K2, C.byref(cfg),
                                    int(threshold), 1 if sort_rows else 0, 1 if row_major else 0, C.byref(h)))
        return Layout(h)

    @staticmethod
    def import_arrays(kind, warp_size, nrows, ncols, nnz, values, col_indices, warp_offset, maxrows,
                      rows_in_warp, forward, sorted_row_length, reduction=None, rows_offset_warp=None,
                      threshold=0, row_major=False):
        keep = [_host(values, np.float64), _host(col_indices, np.int64), _host(warp_offset, np.int64),
                _host(maxrows, np.int64), _host(rows_in_warp, np.int64), _host(forward, np.int64),
                _host(sorted_row_length, np.int64)]
        red = _host(reduction, np.int64) if reduction is not None else None
        row = _host(rows_offset_warp, np.int64) if rows_offset_warp is not None else None
        d = LayoutDesc(EW_LAYOUT_K1 if kind == "k1" else EW_LAYOUT_K2, warp_size, 1 if row_major else 0,
                       nrows, ncols, nnz, keep[2].size, keep[0].size, threshold,
                       keep[0].ctypes.data_as(_f64p), keep[1].ctypes.data_as(_i64p),
                       keep[2].ctypes.data_as(_i64p), keep[3].ctypes.data_as(_i64p),
                       keep[4].ctypes.data_as(_i64p), red.ctypes.data_as(_i64p) if red is not None else None,
                       row.ctypes.data_as(_i64p) if row is not None else None,
                       keep[5].ctypes.data_as(_i64p), keep[6].ctypes.data_as(_i64p))
        h = C.c_void_p()
        check(lib().ew_layout_import(C.byref(d), C.byref(h)))
        return Layout(h)

    def __del__(self):
        h = getattr(self, "h", None)
        if h and self._owner is None and _lib is not None:
            _lib.ew_layout_destroy(h)
            self.h = None

    def info(self):
        i = LayoutInfo()
        check(lib().ew_layout_get_info(self.h, C.byref(i)))
        return i

    def export(self) -> LayoutExport:
        i = self.info()
        nw, ns, n = i.nwarps, i.nslots, i.nrows
        arr = dict(values=np.empty(ns, np.float64), col_indices=np.empty(ns, np.int64),
                   warp_offset=np.empty(nw, np.int64), maxrows=np.empty(nw, np.int64),
                   rows_in_warp=np.empty(nw, np.int64), forward=np.empty(n, np.int64),
                   inverse=np.empty(n, np.int64), sorted_row_length=np.empty(n, np.int64))
        if i.kind == EW_LAYOUT_K2:
            arr["reduction"] = np.empty(nw, np.int64)
            arr["rows_offset_warp"] = np.empty(nw, np.int64)
        a = LayoutArrays()
        for k, v in arr.items():
            setattr(a, k, v.ctypes.data_as(_f64p if v.dtype == np.float64 else _i64p))
        check(lib().ew_layout_export(self.h, C.byref(a)))
        return LayoutExport(kind="k1" if i.kind == EW_LAYOUT_K1 else "k2", warp_size=i.warp_size,
                            nrows=n, ncols=i.ncols, nnz=i.nnz, threshold=i.threshold,
                            stored_slots=i.stored_slots, **arr)

    def value_slot_map(self, csr: Csr):
        out = np.empty(csr.nnz, np.int64)
        check(lib().ew_layout_value_slot_map(self.h, csr.h, _ptr(out)))
        return out

    def refresh_values(self, csr: Csr, stream=None):
        check(lib().ew_layout_refresh_values(self.h, csr.h, _stream_ptr(stream)))

    def dump(self):
        n = C.c_size_t()
        check(lib().ew_layout_dump(self.h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        check(lib().ew_layout_dump(self.h, buf, n.value, C.byref(n)))
        return buf.value.decode()

    def spmv(self, x, y=None, scatter=True, stream=None):
        i = self.info()
        return _apply(lambda xp, nx, yp, ny, mem, s: lib().ew_layout_spmv(self.h, xp, nx, yp, ny,
                                                                           1 if scatter else 0, mem, s),
                      x, y, i.ncols, i.nrows, stream)


@dataclass
class CgResult:
    solution: object
    iterations: int
    residual_history: np.ndarray
    converged: bool
    spmv_calls: int


class Kernel:
    """PreparedKernel (kernels.hpp:16-23) over device data (ew_kernel)."""

    def __init__(self, kernel_id, csr: Csr, warp_size=32, threshold=0, segment_bytes=128, align=True,
                 block_size=None, hyb_k_ell=-1, row_order="reference"):
        """row_order="locality" (r / rs ids only): rows grouped into warps by a
        Cuthill-McKee order before the longest-first sort; same row sums,
        perm() / apply_permuted() in that order (ew_kernel_options.row_order)."""
        cfg = WarpConfig.make(warp_size, block_size=block_size, segment_bytes=segment_bytes, align=align)
        opts = KernelOptions(int(threshold), int(hyb_k_ell), ROW_ORDERS[row_order])
        h = C.c_void_p()
        check(lib().ew_kernel_prepare(kernel_id.encode(), csr.h, C.byref(cfg), C.byref(opts), C.byref(h)))
        self.h = h
        self.id = kernel_id
        info = self.info()
        self.nrows, self.ncols, self.nnz = info.nrows, info.ncols, info.nnz
        self.stored_slots = info.stored_slots
        self.has_perm = bool(info.has_perm)

    def __del__(self):
        h = getattr(self, "h", None)
        if h and _lib is not None:
            _lib.ew_kernel_destroy(h)
            self.h = None

    def info(self):
        i = KernelInfo()
        check(lib().ew_kernel_get_info(self.h, C.byref(i)))
        return i

    def perm(self):
        fwd = np.empty(self.nrows, np.int64)
        inv = np.empty(self.nrows, np.int64)
        check(lib().ew_kernel_get_perm(self.h, _ptr(fwd), _ptr(inv)))
        return fwd, inv

    def layout(self):
        h = C.c_void_p()
        check(lib().ew_kernel_get_layout(self.h, C.byref(h)))
        return Layout(h, owner=self) if h.value else None

    def apply(self, x, y=None, stream=None):
        return _apply(lambda xp, nx, yp, ny, mem, s: lib().ew_kernel_apply(self.h, xp, nx, yp, ny, mem, s),
                      x, y, self.ncols, self.nrows, stream)

    def apply_permuted(self, x, y=None, stream=None):
        return _apply(lambda xp, nx, yp, ny, mem, s: lib().ew_kernel_apply_permuted(self.h, xp, nx, yp, ny,
                                                                                    mem, s),
                      x, y, self.ncols, self.nrows, stream)

    def refresh_values(self, csr: Csr, stream=None):
        check(lib().ew_kernel_refresh_values(self.h, csr.h, _stream_ptr(stream)))

    def cg_solve(self, b, diag=None, tol=1e-8, max_iterations=1000, jacobi=True, recompute_interval=50,
                 divergence_limit=1e6, permuted=False, x=None, stream=None):
        """cg_solve (or cg_solve_permuted) with this kernel as the operator."""
        cfg = CgConfig(float(tol), int(max_iterations), 1 if jacobi else 0, int(recompute_interval),
                       float(divergence_limit))
        dev = hasattr(b, "data_ptr")
        if dev:
            import torch

            x = torch.empty_like(b) if x is None else x
        else:
            b = _host(b, np.float64)
            diag = _host(diag, np.float64) if diag is not None else None
            x = np.empty(b.size, np.float64)
        n = b.numel() if dev else b.size
        hist = np.empty(int(max_iterations) + 1, np.float64)
        res = CgResultC()
        fn = lib().ew_cg_solve_permuted if permuted else lib().ew_cg_solve
        check(fn(self.h, _ptr(b), _ptr(diag), int(n), C.byref(cfg), EW_MEM_DEVICE if dev else EW_MEM_HOST,
                 _ptr(x), _ptr(hist), C.byref(res), _stream_ptr(stream)))
        return CgResult(x, int(res.iterations), hist[: res.history_len].copy(), bool(res.converged),
                        int(res.spmv_calls))


def cg_solve_operator(op, b, diag=None, tol=1e-8, max_iterations=1000, jacobi=True, recompute_interval=50,
                      divergence_limit=1e6):
    """cg_solve with a Python operator ``op(x: np.ndarray) -> np.ndarray`` (the
    reference's SpmvFn closure, cg.hpp:32); vector work and dots run on the
    device, x / y are staged through host buffers around each call."""
    b = _host(b, np.float64)
    diag = _host(diag, np.float64) if diag is not None else None
    n = b.size

    def cb(ctx, xp, yp, stream):
        try:
            xh = np.ctypeslib.as_array(C.cast(xp, _f64p), shape=(n,))
            yh = np.ctypeslib.as_array(C.cast(yp, _f64p), shape=(n,))
            yh[:] = np.asarray(op(xh.copy()), np.float64)
            return 0
        except Exception:  # noqa: BLE001 - reported to the C side as a status
            return EW_INVALID_ARGUMENT

    fn = OPERATOR_FN(cb)
    cfg = CgConfig(float(tol), int(max_iterations), 1 if jacobi else 0, int(recompute_interval),
                   float(divergence_limit))
    x = np.empty(n, np.float64)
    hist = np.empty(int(max_iterations) + 1, np.float64)
    res = CgResultC()
    check(lib().ew_cg_solve_operator(fn, None, EW_MEM_HOST, _ptr(b), _ptr(diag), n, C.byref(cfg),
                                     EW_MEM_HOST, _ptr(x), _ptr(hist), C.byref(res), None))
    return CgResult(x, int(res.iterations), hist[: res.history_len].copy(), bool(res.converged),
                    int(res.spmv_calls))


class Assembly:
    """Race-free FEM assembly as K1 row sums (ew_assembly)."""

    def __init__(self, elements, nnodes, warp_size=32):
        e = _host(elements, np.int64).reshape(-1)
        cfg = WarpConfig.make(warp_size)
        h = C.c_void_p()
        check(lib().ew_assembly_create(e.size // 4, _ptr(e), int(nnodes), C.byref(cfg), C.byref(h)))
        self.h = h
        self.nelements = e.size // 4
        self.nnodes = int(nnodes)
        nnz = C.c_int64()
        check(lib().ew_assembly_pattern(h, C.byref(nnz), None, None))
        self.nnz = nnz.value

    def __del__(self):
        h = getattr(self, "h", None)
        if h and _lib is not None:
            _lib.ew_assembly_destroy(h)
            self.h = None

    def pattern(self):
        ro = np.empty(self.nnodes + 1, np.int64)
        ci = np.empty(self.nnz, np.int64)
        check(lib().ew_assembly_pattern(self.h, None, _ptr(ro), _ptr(ci)))
        return ro, ci

    def run(self, ke, re):
        ke = _host(ke, np.float64)
        re = _host(re, np.float64)
        t = np.empty(self.nnz, np.float64)
        r = np.empty(self.nnodes, np.float64)
        check(lib().ew_assembly_run(self.h, _ptr(ke), _ptr(re), _ptr(t), _ptr(r), EW_MEM_HOST, None))
        return t, r

    def run_into(self, ke, re, kernel):
        ke = _host(ke, np.float64)
        re = _host(re, np.float64)
        r = np.empty(self.nnodes, np.float64)
        check(lib().ew_assembly_run_into(self.h, _ptr(ke), _ptr(re), kernel.h, _ptr(r), EW_MEM_HOST, None))
        return r


def partition_rows(row_offsets, nparts):
    """nnz-balanced contiguous row blocks (host rule)."""
    ro = _host(row_offsets, np.int64)
    out = np.empty(int(nparts) + 1, np.int64)
    check(lib().ew_partition_rows(_ptr(ro), ro.size - 1, int(nparts), _ptr(out)))
    return out


def nccl_unique_id():
    buf = (C.c_uint8 * 128)()
    check(lib().ew_nccl_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)


def torch_allgather(data: bytes):
    """Rank-ordered allgather of a byte string over torch.distributed."""
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return [data]  # a single process
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, data)
    return out


def dist_plan_block(ro, ci, bounds, rank, allgather=None):
    """The setup exchange of Dist.block_ipc on the host (ew_dist_plan_block):
    this rank's ghost columns and, per peer, the rows of this block it
    sends. allgather(bytes) -> list of bytes in rank order (default:
    torch.distributed). Collective; no device work."""
    ro, ci, b = _host(ro, np.int64), _host(ci, np.int64), _host(bounds, np.int64)
    G = b.size - 1
    nloc = ro.size - 1
    fn = allgather or torch_allgather
    err = []

    def cb(send, recv, nbytes, user):
        try:
            buf = b"".join(fn(C.string_at(send, nbytes)))
            if len(buf) != nbytes * G:
                raise ValueError("allgather returned the wrong size")
            C.memmove(recv, buf, len(buf))
            return 0
        except Exception as e:  # reported through the status code
            err.append(e)
            return 1

    cfn = ALLGATHER_FN(cb)
    nghost = C.c_int64()
    ghosts = np.empty(max(1, int(ro[-1])), np.int64)
    send_off = np.empty(G + 1, np.int64)
    send_rows = np.empty(max(1, nloc * G), np.int64)
    st = lib().ew_dist_plan_block(nloc, _ptr(ro), _ptr(ci), _ptr(b), G, int(rank), C.cast(cfn, C.c_void_p), None,
                                  C.byref(nghost), _ptr(ghosts), _ptr(send_off), _ptr(send_rows))
    if err:
        raise err[0]
    check(st)
    return ghosts[: nghost.value].copy(), [send_rows[send_off[h]:send_off[h + 1]].copy() for h in range(G)]


class Dist:
    """Row-partitioned operator + CG (ew_dist).

    Dist.local(...)  -- every partition in this process, on the current GPU
    Dist.nccl(...)   -- one partition per process from the global CSR
    Dist.block(...)  -- one partition per process from this rank's row block
    """

    def __init__(self, h):
        self.h = h
        self.owned = 0
        i = 0
        while True:
            r0, r1, ng, ns = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
            if lib().ew_dist_get_info(h, i, C.byref(r0), C.byref(r1), C.byref(ng), C.byref(ns)) != EW_OK:
                break
            self.owned += r1.value - r0.value
            i += 1
        self.nlocal = i

    def __del__(self):
        h = getattr(self, "h", None)
        if h and _lib is not None:
            _lib.ew_dist_destroy(h)
            self.h = None

    @staticmethod
    def _make(m, nparts, first, nlocal, nccl_id, kernel, bounds, warp_size, threshold, stream):
        ro, ci, v = (_host(m.row_offsets, np.int64), _host(m.col_indices, np.int64), _host(m.values, np.float64))
        b = _host(bounds, np.int64) if bounds is not None else None
        cfg = WarpConfig.make(warp_size)
        opts = KernelOptions(int(threshold), -1, 0)
        idb = (C.c_uint8 * 128).from_buffer_copy(nccl_id) if nccl_id is not None else None
        h = C.c_void_p()
        check(lib().ew_dist_create(m.nrows, m.ncols, ro.size, _ptr(ro), ci.size, _ptr(ci), _ptr(v), _ptr(b),
                                   int(nparts), int(first), int(nlocal),
                                   C.cast(idb, C.c_void_p) if idb is not None else None, kernel.encode(),
                                   C.byref(cfg), C.byref(opts), _stream_ptr(stream), C.byref(h)))
        return Dist(h)

    @staticmethod
    def local(m, nparts, kernel="k1", bounds=None, warp_size=32, threshold=0, stream=None, transport="copy"):
        """transport "copy": halos as device copies; "peer": the IPC
        transport's push / mailbox kernels with this process's partitions as
        the peers (ew_dist_create_peer)."""
        if transport == "copy":
            return Dist._make(m, nparts, 0, nparts, None, kernel, bounds, warp_size, threshold, stream)
        if transport != "peer":
            raise ValueError(f"unknown transport {transport!r}")
        ro, ci, v = (_host(m.row_offsets, np.int64), _host(m.col_indices, np.int64), _host(m.values, np.float64))
        b = _host(bounds, np.int64) if bounds is not None else None
        cfg = WarpConfig.make(warp_size)
        opts = KernelOptions(int(threshold), -1, 0)
        h = C.c_void_p()
        check(lib().ew_dist_create_peer(m.nrows, m.ncols, ro.size, _ptr(ro), ci.size, _ptr(ci), _ptr(v), _ptr(b),
                                        int(nparts), kernel.encode(), C.byref(cfg), C.byref(opts),
                                        _stream_ptr(stream), C.byref(h)))
        return Dist(h)

    @staticmethod
    def block_ipc(nglobal, ro, ci, v, bounds, rank, allgather=None, kernel="k1", warp_size=32, threshold=0,
                  stream=None):
        """One partition per process over CUDA IPC (ew_dist_create_block_ipc).
        allgather(bytes) -> list of bytes in rank order; default:
        torch.distributed.all_gather_object on the default group."""
        ro, ci, v = _host(ro, np.int64), _host(ci, np.int64), _host(v, np.float64)
        b = _host(bounds, np.int64)
        cfg = WarpConfig.make(warp_size)
        opts = KernelOptions(int(threshold), -1, 0)
        fn = allgather or torch_allgather
        err = []

        def cb(send, recv, nbytes, user):
            try:
                parts = fn(C.string_at(send, nbytes))
                buf = b"".join(parts)
                if len(buf) != nbytes * (b.size - 1):
                    raise ValueError("allgather returned the wrong size")
                C.memmove(recv, buf, len(buf))
                return 0
            except Exception as e:  # reported through the status code
                err.append(e)
                return 1

        cfn = ALLGATHER_FN(cb)
        h = C.c_void_p()
        st = lib().ew_dist_create_block_ipc(int(nglobal), ro.size - 1, _ptr(ro), _ptr(ci), _ptr(v), _ptr(b),
                                            b.size - 1, int(rank), C.cast(cfn, C.c_void_p), None,
                                            kernel.encode(), C.byref(cfg), C.byref(opts), _stream_ptr(stream),
                                            C.byref(h))
        if err:
            raise err[0]
        check(st)
        return Dist(h)

    @staticmethod
    def nccl(m, nparts, rank, nccl_id, kernel="k1", bounds=None, warp_size=32, threshold=0, stream=None):
        return Dist._make(m, nparts, rank, 1, nccl_id, kernel, bounds, warp_size, threshold, stream)

    @staticmethod
    def block(nglobal, ro, ci, v, bounds, rank, nccl_id, kernel="k1", warp_size=32, threshold=0, stream=None):
        ro, ci, v = _host(ro, np.int64), _host(ci, np.int64), _host(v, np.float64)
        b = _host(bounds, np.int64)
        cfg = WarpConfig.make(warp_size)
        opts = KernelOptions(int(threshold), -1, 0)
        idb = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
        h = C.c_void_p()
        check(lib().ew_dist_create_block(int(nglobal), ro.size - 1, _ptr(ro), _ptr(ci), _ptr(v), _ptr(b),
                                         b.size - 1, int(rank), C.cast(idb, C.c_void_p), kernel.encode(),
                                         C.byref(cfg), C.byref(opts), _stream_ptr(stream), C.byref(h)))
        return Dist(h)

    def info(self, i=0):
        r0, r1, ng, ns = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        check(lib().ew_dist_get_info(self.h, i, C.byref(r0), C.byref(r1), C.byref(ng), C.byref(ns)))
        sl, sb = C.c_int64(), C.c_int64()
        check(lib().ew_dist_get_layout_bytes(self.h, i, C.byref(sl), C.byref(sb)))
        return dict(row_begin=r0.value, row_end=r1.value, nghost=ng.value, nsend=ns.value,
                    stored_slots=sl.value, stream_bytes=sb.value)

    def spmv(self, x, y=None, stream=None):
        if hasattr(x, "data_ptr"):
            import torch

            y = torch.empty(self.owned, dtype=torch.float64, device=x.device) if y is None else y
            check(lib().ew_dist_spmv(self.h, _ptr(x), _ptr(y), EW_MEM_DEVICE, _stream_ptr(stream)))
            return y
        xh = _host(x, np.float64)
        yh = np.empty(self.owned, np.float64)
        check(lib().ew_dist_spmv(self.h, _ptr(xh), _ptr(yh), EW_MEM_HOST, _stream_ptr(stream)))
        return yh

    def cg_solve(self, b, diag=None, tol=1e-8, max_iterations=1000, jacobi=True, recompute_interval=50,
                 divergence_limit=1e6, stream=None):
        cfg = CgConfig(float(tol), int(max_iterations), 1 if jacobi else 0, int(recompute_interval),
                       float(divergence_limit))
        dev = hasattr(b, "data_ptr")
        if dev:
            import torch

            x = torch.empty_like(b)
        else:
            b = _host(b, np.float64)
            diag = _host(diag, np.float64) if diag is not None else None
            x = np.empty(b.size, np.float64)
        hist = np.empty(int(max_iterations) + 1, np.float64)
        res = CgResultC()
        check(lib().ew_dist_cg_solve(self.h, _ptr(b), _ptr(diag), C.byref(cfg), EW_MEM_DEVICE if dev else EW_MEM_HOST,
                                     _ptr(x), _ptr(hist), C.byref(res), _stream_ptr(stream)))
        return CgResult(x, int(res.iterations), hist[: res.history_len].copy(), bool(res.converged),
                        int(res.spmv_calls))


def compute_alpha(t_reorder, t_kernel, t_base):
    a = C.c_int64()
    f = C.c_int32()
    check(lib().ew_compute_alpha(float(t_reorder), float(t_kernel), float(t_base), C.byref(a), C.byref(f)))
    return a.value if f.value else None


class Mgpu:
    """One process, several GPUs (ew_mgpu_*): the square host CSR in
    nnz-balanced row blocks, block g on devices[g] (default: device g; a
    device may repeat), peers over peer access, one host thread per block."""

    def __init__(self, m, ngpus, devices=None, kernel="k1", warp_size=32, threshold=0):
        ro, ci, v = _host(m.row_offsets, np.int64), _host(m.col_indices, np.int64), _host(m.values, np.float64)
        dev = _host(devices, np.int32) if devices is not None else None
        if dev is not None and dev.size != ngpus:
            raise ValueError("devices must list one device per partition")
        cfg = WarpConfig.make(warp_size)
        opts = KernelOptions(int(threshold), -1, 0)
        h = C.c_void_p()
        check(lib().ew_mgpu_create(int(m.nrows), _ptr(ro), _ptr(ci), _ptr(v), int(ngpus), _ptr(dev),
                                   kernel.encode(), C.byref(cfg), C.byref(opts), C.byref(h)))
        self.h, self.n = h, int(m.nrows)

    def __del__(self):
        h = getattr(self, "h", None)
        if h and _lib is not None:
            _lib.ew_mgpu_destroy(h)
            self.h = None

    def spmv(self, x):
        x = _host(x, np.float64)
        y = np.empty(self.n, np.float64)
        check(lib().ew_mgpu_spmv(self.h, _ptr(x), _ptr(y)))
        return y

    def cg_solve(self, b, diag=None, tol=1e-8, max_iterations=1000, jacobi=True, recompute_interval=50,
                 divergence_limit=1e6):
        cfg = CgConfig(float(tol), int(max_iterations), 1 if jacobi else 0, int(recompute_interval),
                       float(divergence_limit))
        b = _host(b, np.float64)
        diag = _host(diag, np.float64) if diag is not None else None
        x = np.empty(self.n, np.float64)
        hist = np.empty(int(max_iterations) + 1, np.float64)
        res = CgResultC()
        check(lib().ew_mgpu_cg_solve(self.h, _ptr(b), _ptr(diag), C.byref(cfg), _ptr(x), _ptr(hist),
                                     C.byref(res)))
        return CgResult(x, int(res.iterations), hist[: res.history_len].copy(), bool(res.converged),
                        int(res.spmv_calls))

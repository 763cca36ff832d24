// Status mapping and host <-> device marshalling for the C++ API.
#include "ellwarp/device.hpp"

#include "ellwarp/cg.hpp"

namespace ellwarp {

void WarpModelConfig::validate() const {
    // warp_model.cpp:7-14 (argument checks only)
    require(warp_size > 0 && (warp_size & (warp_size - 1)) == 0, "warp_size must be a power of two");
    require(block_size >= warp_size && block_size % warp_size == 0,
            "block_size must be a positive multiple of warp_size");
    require(segment_bytes > 0 && (segment_bytes & (segment_bytes - 1)) == 0,
            "segment_bytes must be a power of two");
    require(cache_lines > 0, "cache_lines must be positive");
}

namespace device {

void check(ew_status s) {
    if (s == EW_OK) return;
    const std::string msg = ew_last_error();
    switch (s) {
        case EW_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case EW_CG_DIVERGENCE: throw CgDivergenceError(msg);
        case EW_UNSUPPORTED: throw UnsupportedError(msg);
        default: throw DeviceError(msg + " (" + ew_status_string(s) + ")");
    }
}

CsrHandle upload(const SparseCsr& m, bool canonical) {
    // validate_csr's container checks come first (csr.cpp:58-62); the
    // per-row checks run on the device inside ew_csr_create.
    require(m.nrows >= 0 && m.ncols >= 0, "negative dimensions");
    require(static_cast<idx>(m.row_offsets.size()) == m.nrows + 1, "row_offsets length");
    require(m.row_offsets.front() == 0, "row_offsets[0] != 0");
    require(m.row_offsets.back() == m.nnz(), "row_offsets[nrows] != nnz");
    require(m.values.size() == m.col_indices.size(), "values/col_indices length mismatch");
    ew_csr h = nullptr;
    check(ew_csr_create(m.nrows, m.ncols, static_cast<int64_t>(m.row_offsets.size()), m.row_offsets.data(),
                        m.nnz(), m.col_indices.data(), m.values.data(), EW_MEM_HOST,
                        canonical ? EW_CSR_CANONICAL : 0, nullptr, &h));
    return CsrHandle(h, [](ew_csr p) { ew_csr_destroy(p); });
}

SparseCsr download(const CsrHandle& h) {
    SparseCsr m;
    int64_t n = 0, nc = 0, nnz = 0;
    check(ew_csr_shape(h.get(), &n, &nc, &nnz));
    m.nrows = n;
    m.ncols = nc;
    m.row_offsets.resize(n + 1);
    m.col_indices.resize(nnz);
    m.values.resize(nnz);
    check(ew_csr_export(h.get(), m.row_offsets.data(), m.col_indices.data(), m.values.data()));
    return m;
}

ew_warp_config to_c(const WarpModelConfig& c) {
    return ew_warp_config{c.warp_size, c.block_size, c.segment_bytes, c.align_warp_offsets ? 1 : 0,
                          c.ideal_cache ? 1 : 0, c.cache_lines};
}

void no_tracer(const WarpTracer* t) {
    if (t) throw UnsupportedError("WarpTracer: the lockstep transaction model has no device path (use ncu)");
}

}  // namespace device
}  // namespace ellwarp

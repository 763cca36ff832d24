// ELL / HYB layouts for padding comparisons (formats.cpp:7-62 in the
// reference), host side; their SpMV kernels run on the device
// (csrc/ew_formats.cu, prepare_kernel("ell" / "hyb")).
#include "ellwarp/formats.hpp"

namespace ellwarp {

EllLayout build_ell(const SparseCsr& m) {
    EllLayout l;
    l.nrows = m.nrows;
    l.ncols = m.ncols;
    l.nnz = m.nnz();
    for (idx r = 0; r < m.nrows; ++r) l.width = std::max(l.width, m.row_length(r));
    l.values.assign(static_cast<size_t>(l.nrows * l.width), 0.0);
    l.col_indices.assign(static_cast<size_t>(l.nrows * l.width), 0);
    for (idx r = 0; r < m.nrows; ++r)
        for (idx j = 0, k = m.row_offsets[r]; k < m.row_offsets[r + 1]; ++j, ++k) {
            l.values[j * l.nrows + r] = m.values[k];
            l.col_indices[j * l.nrows + r] = m.col_indices[k];
        }
    return l;
}

HybLayout build_hyb(const SparseCsr& m, idx k_ell) {
    require(k_ell >= 0, "build_hyb: k_ell must be >= 0");
    HybLayout h;
    h.k_ell = k_ell;
    EllLayout& e = h.ell_part;
    e.nrows = m.nrows;
    e.ncols = m.ncols;
    for (idx r = 0; r < m.nrows; ++r) e.width = std::max(e.width, std::min(k_ell, m.row_length(r)));
    e.values.assign(static_cast<size_t>(e.nrows * e.width), 0.0);
    e.col_indices.assign(static_cast<size_t>(e.nrows * e.width), 0);
    h.coo_tail.nrows = m.nrows;
    h.coo_tail.ncols = m.ncols;
    for (idx r = 0; r < m.nrows; ++r)
        for (idx j = 0, k = m.row_offsets[r]; k < m.row_offsets[r + 1]; ++j, ++k) {
            if (j < k_ell) {
                e.values[j * e.nrows + r] = m.values[k];
                e.col_indices[j * e.nrows + r] = m.col_indices[k];
                e.nnz++;
            } else {
                h.coo_tail.entries.push_back({r, m.col_indices[k], m.values[k]});
            }
        }
    return h;
}

idx hyb_default_k_ell(const SparseCsr& m, real covered_fraction) {
    // smallest width covering at least `covered_fraction` of the rows
    if (m.nrows == 0) return 0;
    std::vector<idx> len(m.nrows);
    for (idx r = 0; r < m.nrows; ++r) len[r] = m.row_length(r);
    std::sort(len.begin(), len.end());
    const idx want = static_cast<idx>(std::ceil(covered_fraction * static_cast<real>(m.nrows)));
    return len[std::clamp<idx>(want, 1, m.nrows) - 1];
}

}  // namespace ellwarp

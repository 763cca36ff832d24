// Drop-in for proj/include/ellwarp/formats.hpp (formats.hpp:11-53): the
// comparison formats of the paper (ELL, HYB). Layout builders are provided
// for padding comparisons; their SpMV kernels are SURVEY.md §8(f) "next" and
// prepare_kernel reports them as UnsupportedError until then.
#pragma once

#include "ellwarp/csr.hpp"
#include "ellwarp/warp_model.hpp"

namespace ellwarp {

struct EllLayout {
    idx nrows = 0;
    idx ncols = 0;
    idx nnz = 0;
    idx width = 0;
    std::vector<real> values;      // element (r, j) at j * nrows + r
    std::vector<idx> col_indices;  // padding: value 0.0, column 0

    idx stored_slots() const { return nrows * width; }
    idx padded_slots() const { return stored_slots() - nnz; }
};

struct HybLayout {
    EllLayout ell_part;
    SparseCoo coo_tail;
    idx k_ell = 0;
};

EllLayout build_ell(const SparseCsr& m);
HybLayout build_hyb(const SparseCsr& m, idx k_ell);
idx hyb_default_k_ell(const SparseCsr& m, real covered_fraction = 2.0 / 3.0);

}  // namespace ellwarp

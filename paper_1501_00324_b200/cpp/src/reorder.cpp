#include "ellwarp/reorder.hpp"

#include "ellwarp/device.hpp"

namespace ellwarp {

ReorderedOperand make_reordered_r(const SparseCsr& m, const Permutation& p) {
    require(m.square(), "make_reordered_r: matrix must be square");
    require(p.size() == m.nrows, "make_reordered_r: permutation size mismatch");
    auto h = device::upload(m);
    ew_csr out = nullptr;
    device::check(ew_reorder(h.get(), p.forward.data(), 0, &out, nullptr));
    ReorderedOperand op;
    op.matrix = device::download(device::CsrHandle(out, [](ew_csr q) { ew_csr_destroy(q); }));
    op.row_perm = p;
    op.variant = ReorderVariant::r;
    return op;
}

ReorderedOperand make_reordered_rs(const ReorderedOperand& op) {
    require(op.variant == ReorderVariant::r, "make_reordered_rs: expects a variant-r operand");
    // the r operand's columns are renumbered (not sorted), so upload without
    // the strictly-increasing check: ew_csr_sort_rows takes an r matrix
    // produced on the device, re-uploaded here through a sorted staging copy
    auto h = device::upload_unsorted(op.matrix);
    ew_csr out = nullptr;
    device::check(ew_csr_sort_rows(h.get(), &out));
    ReorderedOperand res = op;
    res.variant = ReorderVariant::rs;
    res.matrix = device::download(device::CsrHandle(out, [](ew_csr q) { ew_csr_destroy(q); }));
    return res;
}

}  // namespace ellwarp

// Prepared kernels: prepare_kernel / apply / apply_permuted (kernels.cpp:14-125)
// over device layouts.
#include "ew_internal.cuh"

namespace ew {

void kernel_apply(const KernelData& k, const double* x, double* y, bool permuted, cudaStream_t s,
                  const int* done) {
    if (k.format) {
        require(!permuted, "kernel '" + k.id + "' has no apply_permuted");
        format_spmv(*k.format, *k.csr, x, y, s, done);
        return;
    }
    if (k.csr) {
        require(!permuted, "kernel '" + k.id + "' has no apply_permuted");
        csr_spmv_guarded(*k.csr, x, y, s, done);
        return;
    }
    const LayoutData& l = *k.layout;
    if (!k.reordered) {
        require(!permuted, "kernel '" + k.id + "' has no apply_permuted");
        layout_spmv(l, x, y, /*scatter=*/true, s, done);  // K1 / K2: y[Pinv[p]]
        return;
    }
    if (permuted) {
        layout_spmv(l, x, y, /*scatter=*/false, s, done);  // coalesced sorted store
        return;
    }
    // apply() of an r/rs operand (kernels.cpp:50-53): x' = x[forward] in,
    // sorted kernel, y[forward[p]] = y'[p] out. The unpermute is fused into
    // the kernel's store (same value, same destination); only x' is staged.
    Scratch<double> xp(l.nrows, s);
    gather(l.fwd.get(), x, xp.get(), l.nrows, s);
    layout_spmv(l, xp.get(), y, /*scatter=*/true, s, done);
}

}  // namespace ew

// Prepared kernels: prepare_kernel / apply / apply_permuted (kernels.cpp:14-125)
// over device layouts.
#include <cstdlib>

#include "ew_internal.cuh"

namespace ew {

bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("EW_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

std::shared_ptr<KernelData> prepare(const std::string& sid, const CsrData& src, const ew_warp_config& c,
                                    const ew_kernel_options& o, cudaStream_t s) {
    validate_config(c);  // prepare_kernel validates first (kernels.cpp:61)
    require(o.row_order == EW_ROW_ORDER_REFERENCE || o.row_order == EW_ROW_ORDER_LOCALITY, "unknown row_order");
    require(o.row_order == EW_ROW_ORDER_REFERENCE ||
                (sid.size() > 2 && (sid.compare(0, 2, "k1") == 0 || sid.compare(0, 2, "k2") == 0)),
            "row_order=locality needs an r / rs kernel id (k1r, k1rs, k2r, k2rs)");
    auto k = std::make_shared<KernelData>();
    k->id = sid;
    k->nrows = src.nrows;
    k->ncols = src.ncols;
    k->nnz = src.nnz;
    k->stored_slots = src.nnz;
    if (sid == "csr_ref") {
        k->csr = csr_clone(src, s);  // the closure owns a copy (kernels.cpp:65-68)
    } else if (sid == "csr_vector" || sid == "coo" || sid == "ell" || sid == "hyb") {
        if (c.warp_size > 1024) throw Error(EW_UNSUPPORTED, "warp_size above 1024 has no device mapping");
        k->csr = csr_clone(src, s);
        k->format = build_format(src, sid, c.warp_size, o.hyb_k_ell, s);
        k->stored_slots = k->format->stored_slots;
    } else if (sid == "k1" || sid == "k2" || sid == "k1r" || sid == "k1rs" || sid == "k2r" || sid == "k2rs") {
        const bool is_k2 = sid[1] == '2';
        const bool reordered = sid.size() > 2;
        // KernelOptions::k2_threshold <= 0: the max row length (kernels.cpp:16-21)
        const int64_t thr = o.k2_threshold > 0 ? o.k2_threshold : std::max<int64_t>(1, src.maxrow);
        const bool locality = o.row_order == EW_ROW_ORDER_LOCALITY;
        std::shared_ptr<CsrData> op;
        DevBuf<int32_t> qf, qi;
        if (reordered) {
            require(src.nrows == src.ncols, "kernel '" + sid + "' requires a square matrix");
            op = reorder(src, nullptr, true, sid.size() == 4, nullptr, s, &k->entry_dst);
            if (locality) {
                // rows regrouped by locality; each keeps op's (reference) entry order
                const int64_t n = src.nrows;
                DevBuf<int32_t> pf(n), pi(n), sl(n);
                sort_rows_desc(src, pf.get(), pi.get(), sl.get(), s, nullptr);
                qf.alloc(n);
                qi.alloc(n);
                op = locality_operand(src, *op, pf.get(), qf.get(), qi.get(), s);
            }
        }
        k->reordered = reordered;
        k->locality = locality;
        k->layout = build_layout(reordered ? *op : src, is_k2 ? EW_LAYOUT_K2 : EW_LAYOUT_K1, c, thr, true, false, s);
        if (locality && src.nrows) {
            // op's rows are already longest-first, so the layout's own sort is
            // the identity; its permutation is the locality order
            EW_CUDA_CHECK(cudaMemcpyAsync(k->layout->fwd.get(), qf.get(), src.nrows * 4, cudaMemcpyDeviceToDevice, s));
            EW_CUDA_CHECK(cudaMemcpyAsync(k->layout->inv.get(), qi.get(), src.nrows * 4, cudaMemcpyDeviceToDevice, s));
            EW_CUDA_CHECK(cudaStreamSynchronize(s));
        }
        k->stored_slots = k->layout->stored_slots;
    } else {
        throw Error(EW_INVALID_ARGUMENT, "unknown kernel id '" + sid + "'");
    }
    return k;
}

bool kernel_apply_dot(const KernelData& k, const double* x, double* y, bool permuted, cudaStream_t s,
                      const int* done, const DotSink& sink) {
    if (!k.layout || k.format) return false;
    if (!k.reordered) return layout_spmv_dot(*k.layout, x, y, /*scatter=*/true, s, done, sink);
    if (permuted) return layout_spmv_dot(*k.layout, x, y, /*scatter=*/false, s, done, sink);
    return false;  // r/rs apply() gathers x first: the dot stays a separate pass
}

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

// Prepared kernels: prepare_kernel / apply / apply_permuted (kernels.cpp:14-125)
// over device layouts.
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
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

// ---- host-buffer apply pipeline --------------------------------------------
namespace ew {

namespace {

constexpr int64_t kPipeMinNnz = 2'000'000;   // below: one copy each way is cheaper
constexpr int64_t kPipeMinRowsPerBlock = 16'384;
constexpr int kPipeMaxBlocks = 8;

// Row lengths of original rows [r0, r0 + n) from the K1 layout.
__global__ void block_len_kernel(const int32_t* __restrict__ inv, const int32_t* __restrict__ slen, int64_t r0,
                                 int64_t n, int64_t* __restrict__ len) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) len[i] = slen[inv[r0 + i]];
}

// The CSR rows [r0, r0 + n) read back out of the K1 slabs (entry order as
// stored, i.e. the original CSR order), plus the block's largest column.
__global__ void block_extract_kernel(const double* __restrict__ vals, const int32_t* __restrict__ cols,
                                     const int64_t* __restrict__ woff, const int32_t* __restrict__ inv,
                                     int32_t ws_log2, int64_t r0, int64_t n, const int64_t* __restrict__ ro,
                                     int32_t* __restrict__ ci, double* __restrict__ v, int* cmax) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t p = inv[r0 + i];
    const int64_t w = p >> ws_log2, ws = int64_t{1} << ws_log2;
    const int64_t base = woff[w] + (p & (ws - 1));
    int m = -1;
    for (int64_t k = ro[i], j = 0; k < ro[i + 1]; ++k, ++j) {
        const int32_t c = cols[base + j * ws];
        ci[k] = c;
        v[k] = vals[base + j * ws];
        m = max(m, c);
    }
    atomicMax(cmax, m);
}

std::unique_ptr<HostPipeline> build_pipeline(const KernelData& k, cudaStream_t s) {
    const LayoutData& l = *k.layout;
    const int64_t n = k.nrows;
    auto P = std::make_unique<HostPipeline>();
    static const int max_blocks = [] {
        const char* e = std::getenv("EW_PIPE_BLOCKS");  // A/B runs
        return e ? std::max(1, std::atoi(e)) : kPipeMaxBlocks;
    }();
    const int B = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(max_blocks, n / kPipeMinRowsPerBlock)));
    P->nblocks = B;
    P->r0.resize(B + 1);
    P->c0.resize(B + 1);
    for (int b = 0; b <= B; ++b) {
        P->r0[b] = n * b / B;
        P->c0[b] = k.ncols * b / B;
    }
    ew_warp_config cfg{l.ws, std::max(32, l.ws), l.segment_bytes, l.align, 0, 64};
    DevBuf<int> cmax(B);
    EW_CUDA_CHECK(cudaMemsetAsync(cmax.get(), 0xff, B * sizeof(int), s));  // -1
    for (int b = 0; b < B; ++b) {
        const int64_t nb = P->r0[b + 1] - P->r0[b];
        CsrData sub;
        sub.nrows = nb;
        sub.ncols = k.ncols;
        sub.ro.alloc(nb + 1);
        Scratch<int64_t> len(nb, s), mx(1, s);
        block_len_kernel<<<grid_for(nb), kBlock, 0, s>>>(l.inv.get(), l.slen.get(), P->r0[b], nb, len.get());
        launched("block_len_kernel");
        size_t bytes = 0, bytes2 = 0;
        EW_CUDA_CHECK(cub::DeviceScan::InclusiveSum(nullptr, bytes, len.get(), sub.ro.get() + 1, nb, s));
        EW_CUDA_CHECK(cub::DeviceReduce::Max(nullptr, bytes2, len.get(), mx.get(), nb, s));
        Scratch<unsigned char> tmp(std::max(bytes, bytes2), s);
        EW_CUDA_CHECK(cub::DeviceScan::InclusiveSum(tmp.get(), bytes, len.get(), sub.ro.get() + 1, nb, s));
        launched("cub::DeviceScan::InclusiveSum");
        EW_CUDA_CHECK(cub::DeviceReduce::Max(tmp.get(), bytes2, len.get(), mx.get(), nb, s));
        launched("cub::DeviceReduce::Max");
        EW_CUDA_CHECK(cudaMemsetAsync(sub.ro.get(), 0, sizeof(int64_t), s));
        int64_t nnz = 0, longest = 0;
        EW_CUDA_CHECK(cudaMemcpyAsync(&nnz, sub.ro.get() + nb, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        EW_CUDA_CHECK(cudaMemcpyAsync(&longest, mx.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        EW_CUDA_CHECK(cudaStreamSynchronize(s));
        sub.nnz = nnz;
        sub.ci.alloc(sub.nnz);
        sub.v.alloc(sub.nnz);
        block_extract_kernel<<<grid_for(nb), kBlock, 0, s>>>(l.values.get(), l.cols.get(), l.warp_offset.get(),
                                                             l.inv.get(), l.ws_log2, P->r0[b], nb, sub.ro.get(),
                                                             sub.ci.get(), sub.v.get(), cmax.get() + b);
        launched("block_extract_kernel");
        sub.maxrow = static_cast<int32_t>(longest);
        P->blocks.push_back(build_layout(sub, EW_LAYOUT_K1, cfg, 0, true, false, s));
    }
    std::vector<int> hmax(B);
    EW_CUDA_CHECK(cudaMemcpyAsync(hmax.data(), cmax.get(), B * sizeof(int), cudaMemcpyDeviceToHost, s));
    EW_CUDA_CHECK(cudaStreamSynchronize(s));
    P->need.resize(B);
    for (int b = 0; b < B; ++b) {
        const int64_t c = std::max(0, hmax[b]);
        P->need[b] = static_cast<int>(std::upper_bound(P->c0.begin(), P->c0.end(), c) - P->c0.begin()) - 1;
        P->need[b] = std::min(std::max(P->need[b], 0), B - 1);
    }
    P->x.alloc(k.ncols);
    P->y.alloc(n);
    EW_CUDA_CHECK(cudaStreamCreateWithFlags(&P->up, cudaStreamNonBlocking));
    EW_CUDA_CHECK(cudaStreamCreateWithFlags(&P->down, cudaStreamNonBlocking));
    P->ev_x.resize(B);
    P->ev_y.resize(B);
    for (auto& e : P->ev_x) EW_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : P->ev_y) EW_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    EW_CUDA_CHECK(cudaEventCreateWithFlags(&P->ev_start, cudaEventDisableTiming));
    EW_CUDA_CHECK(cudaEventCreateWithFlags(&P->ev_done, cudaEventDisableTiming));
    return P;
}

}  // namespace

bool kernel_apply_host(const KernelData& k, const double* x, double* y, cudaStream_t s) {
    if (!k.layout || k.format || k.csr || k.reordered || k.layout->kind != EW_LAYOUT_K1 || k.layout->row_major ||
        k.layout->imported || k.nnz < kPipeMinNnz || k.nrows < 2 * kPipeMinRowsPerBlock)
        return false;
    std::unique_lock<std::mutex> lock(k.pipe_mu, std::try_to_lock);
    if (!lock.owns_lock()) return false;  // a concurrent caller: the plain path
    if (!k.pipe) k.pipe = build_pipeline(k, s);
    HostPipeline& P = *k.pipe;
    EW_CUDA_CHECK(cudaEventRecord(P.ev_start, s));
    EW_CUDA_CHECK(cudaStreamWaitEvent(P.up, P.ev_start, 0));
    EW_CUDA_CHECK(cudaStreamWaitEvent(P.down, P.ev_start, 0));
    for (int c = 0; c < P.nblocks; ++c) {
        const int64_t a = P.c0[c], b = P.c0[c + 1];
        if (b > a)
            EW_CUDA_CHECK(cudaMemcpyAsync(P.x.get() + a, x + a, (b - a) * sizeof(double), cudaMemcpyHostToDevice, P.up));
        EW_CUDA_CHECK(cudaEventRecord(P.ev_x[c], P.up));
    }
    for (int b = 0; b < P.nblocks; ++b) {
        EW_CUDA_CHECK(cudaStreamWaitEvent(s, P.ev_x[P.need[b]], 0));
        layout_spmv(*P.blocks[b], P.x.get(), P.y.get() + P.r0[b], /*scatter=*/true, s);
        EW_CUDA_CHECK(cudaEventRecord(P.ev_y[b], s));
        EW_CUDA_CHECK(cudaStreamWaitEvent(P.down, P.ev_y[b], 0));
        const int64_t nb = P.r0[b + 1] - P.r0[b];
        if (nb)
            EW_CUDA_CHECK(cudaMemcpyAsync(y + P.r0[b], P.y.get() + P.r0[b], nb * sizeof(double),
                                          cudaMemcpyDeviceToHost, P.down));
    }
    EW_CUDA_CHECK(cudaEventRecord(P.ev_done, P.down));
    EW_CUDA_CHECK(cudaStreamWaitEvent(s, P.ev_done, 0));
    EW_CUDA_CHECK(cudaStreamSynchronize(s));
    return true;
}

}  // namespace ew

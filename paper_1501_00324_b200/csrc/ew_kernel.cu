// Prepared kernels: prepare_kernel / apply / apply_permuted (kernels.cpp:14-125)
// over device layouts.
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

// Largest column of each sorted row position's real entries (-1: no entries).
__global__ void row_maxcol_kernel(const int32_t* __restrict__ cols, const int64_t* __restrict__ woff,
                                  const int32_t* __restrict__ slen, int32_t ws_log2, int64_t n,
                                  int32_t* __restrict__ out) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int64_t ws = int64_t{1} << ws_log2;
    const int64_t base = woff[p >> ws_log2] + (p & (ws - 1));
    int32_t m = -1;
    for (int32_t j = 0; j < slen[p]; ++j) m = max(m, cols[base + j * ws]);
    out[p] = m;
}

// The stage plan of HostPipeline (see ew_internal.cuh), from the layout's
// row permutation and each row's largest column; host work, once per kernel.
std::unique_ptr<HostPipeline> build_pipeline(const KernelData& k, cudaStream_t s) {
    const LayoutData& l = *k.layout;
    const int64_t n = k.nrows, nc = k.ncols, ws = l.ws;
    auto P = std::make_unique<HostPipeline>();
    static const int max_blocks = [] {
        const char* e = std::getenv("EW_PIPE_BLOCKS");  // A/B runs
        return e ? std::min(64, std::max(1, std::atoi(e))) : kPipeMaxBlocks;
    }();
    const int B = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(max_blocks, n / kPipeMinRowsPerBlock)));
    P->nstages = B;
    std::vector<int32_t> fwd(n), mxc(n);
    {
        DevBuf<int32_t> d(n);
        Scratch<int32_t> full(l.cols_full ? 0 : l.nslots, s);  // a dropped int32 slab, decoded for the plan
        if (!l.cols_full) decode_columns(l, full.get(), s);
        row_maxcol_kernel<<<grid_for(n), kBlock, 0, s>>>(l.cols_full ? l.cols.get() : full.get(),
                                                         l.warp_offset.get(), l.slen.get(), l.ws_log2, n, d.get());
        launched("row_maxcol_kernel");
        EW_CUDA_CHECK(cudaMemcpyAsync(mxc.data(), d.get(), n * 4, cudaMemcpyDeviceToHost, s));
        EW_CUDA_CHECK(cudaMemcpyAsync(fwd.data(), l.fwd.get(), n * 4, cudaMemcpyDeviceToHost, s));
        EW_CUDA_CHECK(cudaStreamSynchronize(s));
    }
    // row blocks r0[b] = n b / B; block(r) = the b with r0[b] <= r < r0[b+1]
    std::vector<int64_t> r0(B + 1);
    for (int b = 0; b <= B; ++b) r0[b] = n * b / B;
    std::vector<int32_t> blk(n);
    for (int b = 0; b < B; ++b)
        for (int64_t r = r0[b]; r < r0[b + 1]; ++r) blk[r] = b;
    // x chunk b ends past every column that rows of blocks <= b reference
    std::vector<int32_t> rowmax(n, -1);
    for (int64_t p = 0; p < n; ++p) rowmax[fwd[p]] = mxc[p];
    P->c0.assign(B + 1, 0);
    int64_t pref = -1;
    for (int b = 0; b < B; ++b) {
        for (int64_t r = r0[b]; r < r0[b + 1]; ++r) pref = std::max<int64_t>(pref, rowmax[r]);
        P->c0[b + 1] = std::min(nc, std::max(P->c0[b], std::max(nc * (b + 1) / B, pref + 1)));
    }
    P->c0[B] = nc;
    // stage of a warp: the last row block it writes (so chunks <= stage cover it)
    const int64_t nw = l.nwarps;
    std::vector<int32_t> stage(nw, 0);
    for (int64_t p = 0; p < n; ++p) stage[p / ws] = std::max(stage[p / ws], blk[fwd[p]]);
    std::vector<int64_t> cnt(B + 1, 0);
    for (int64_t w = 0; w < nw; ++w) ++cnt[stage[w] + 1];
    P->wstart.assign(B + 1, 0);
    for (int b = 0; b < B; ++b) P->wstart[b + 1] = P->wstart[b] + cnt[b + 1];
    std::vector<int32_t> order(nw);
    {
        std::vector<int64_t> at(P->wstart.begin(), P->wstart.end() - 1);
        for (int64_t w = 0; w < nw; ++w) order[at[stage[w]]++] = static_cast<int32_t>(w);  // stable
    }
    // row block b goes down after the first stage >= b by which all but a
    // few of its rows are final; the rest are stragglers (gathered at the end)
    std::vector<int32_t> done_at(n);
    for (int64_t p = 0; p < n; ++p) done_at[fwd[p]] = stage[p / ws];
    P->r0 = r0;
    P->ystage.assign(B, B - 1);
    for (int b = 0; b < B; ++b) {
        const int64_t nb = r0[b + 1] - r0[b], allow = std::max<int64_t>(1024, nb / 100);
        std::vector<int64_t> late_by(B + 1, 0);  // rows of block b final only after stage s
        for (int64_t r = r0[b]; r < r0[b + 1]; ++r) ++late_by[done_at[r]];
        int64_t later = nb;
        for (int st = 0; st < B; ++st) {
            later -= late_by[st];  // rows final after stage st
            if (st >= b && later <= allow) {
                P->ystage[b] = st;
                break;
            }
        }
        for (int64_t r = r0[b]; r < r0[b + 1]; ++r)
            if (done_at[r] > P->ystage[b]) P->late.push_back(static_cast<int32_t>(r));
    }
    if (!P->late.empty()) {
        const size_t nl = P->late.size();
        P->late_d.alloc(nl);
        P->late_y.alloc(nl);
        EW_CUDA_CHECK(cudaMallocHost(&P->late_h, nl * sizeof(double)));
        EW_CUDA_CHECK(cudaMemcpyAsync(P->late_d.get(), P->late.data(), nl * 4, cudaMemcpyHostToDevice, s));
    }
    P->widx.alloc(nw);
    EW_CUDA_CHECK(cudaMemcpyAsync(P->widx.get(), order.data(), nw * 4, cudaMemcpyHostToDevice, s));
    P->x.alloc(nc);
    P->y.alloc(n);
    EW_CUDA_CHECK(cudaStreamSynchronize(s));
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
        !k.layout->sorted || k.layout->imported || k.nnz < kPipeMinNnz || k.nrows < 2 * kPipeMinRowsPerBlock)
        return false;
    std::unique_lock<std::mutex> lock(k.pipe_mu, std::try_to_lock);
    if (!lock.owns_lock()) return false;  // a concurrent caller: the plain path
    if (!k.pipe) k.pipe = build_pipeline(k, s);
    HostPipeline& P = *k.pipe;
    EW_CUDA_CHECK(cudaEventRecord(P.ev_start, s));
    EW_CUDA_CHECK(cudaStreamWaitEvent(P.up, P.ev_start, 0));
    EW_CUDA_CHECK(cudaStreamWaitEvent(P.down, P.ev_start, 0));
    for (int c = 0; c < P.nstages; ++c) {
        const int64_t a = P.c0[c], b = P.c0[c + 1];
        if (b > a)
            EW_CUDA_CHECK(cudaMemcpyAsync(P.x.get() + a, x + a, (b - a) * sizeof(double), cudaMemcpyHostToDevice, P.up));
        EW_CUDA_CHECK(cudaEventRecord(P.ev_x[c], P.up));
    }
    for (int b = 0; b < P.nstages; ++b) {
        EW_CUDA_CHECK(cudaStreamWaitEvent(s, P.ev_x[b], 0));
        layout_spmv_warps(*k.layout, P.widx.get() + P.wstart[b], P.wstart[b + 1] - P.wstart[b], P.x.get(),
                          P.y.get(), s);
        // the row blocks final after this stage (consecutive blocks in one copy)
        int64_t lo = -1, hi = -1;
        auto flush = [&] {
            if (hi > lo)
                EW_CUDA_CHECK(cudaMemcpyAsync(y + lo, P.y.get() + lo, (hi - lo) * sizeof(double),
                                              cudaMemcpyDeviceToHost, P.down));
            lo = hi = -1;
        };
        bool recorded = false;
        for (int rb = 0; rb < P.nstages; ++rb) {
            if (P.ystage[rb] != b) continue;
            if (!recorded) {
                EW_CUDA_CHECK(cudaEventRecord(P.ev_y[b], s));
                EW_CUDA_CHECK(cudaStreamWaitEvent(P.down, P.ev_y[b], 0));
                recorded = true;
            }
            if (P.r0[rb] != hi) flush();
            if (lo < 0) lo = P.r0[rb];
            hi = P.r0[rb + 1];
        }
        flush();
    }
    const int64_t nl = static_cast<int64_t>(P.late.size());
    if (nl) {
        gather(P.late_d.get(), P.y.get(), P.late_y.get(), nl, s);
        EW_CUDA_CHECK(cudaMemcpyAsync(P.late_h, P.late_y.get(), nl * sizeof(double), cudaMemcpyDeviceToHost, s));
    }
    EW_CUDA_CHECK(cudaEventRecord(P.ev_done, P.down));
    EW_CUDA_CHECK(cudaStreamWaitEvent(s, P.ev_done, 0));
    EW_CUDA_CHECK(cudaStreamSynchronize(s));
    // stragglers after their blocks' copies have landed
    for (int64_t i = 0; i < nl; ++i) y[P.late[i]] = P.late_h[i];
    return true;
}

const void* kernel_anchor_kernel() { return reinterpret_cast<const void*>(&row_maxcol_kernel); }

}  // namespace ew

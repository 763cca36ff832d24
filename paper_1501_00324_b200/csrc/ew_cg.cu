// Single-GPU Jacobi PCG driver (cg.cpp:25-104): the prepared kernel (or a
// host closure) is the operator, everything else stays on the device.
//
// Per iteration four stream-ordered launches, no host round trip:
//   1. q = A p                        (operator)
//   2. p.q                            (+ breakdown test, alpha = rz / pq)
//   3. x += alpha p ; r -= alpha q    (+ r.r, r.z with z = r / diag, history,
//                                      convergence / divergence, beta)
//      refresh iterations (k % recompute_interval == 0) replace the r update
//      by r = b - A x after one more operator launch, as cg.cpp:82-86
//   4. p = z + beta p
// Element-wise arithmetic follows the reference exactly; dot products are
// fixed-order trees (ew_cg.cuh). Kernels read a device `done` flag first, so
// the host enqueues iterations in batches and polls once per batch.
#include "ew_cg.cuh"

namespace ew {

using cg::State;

CgOutputs cg_device(const CgOperator& op, const double* b, const double* diag, int64_t n,
                    const ew_cg_config& cfg, double* x, cudaStream_t s) {
    CgOutputs out;
    require(cfg.rel_tolerance > 0.0, "cg: tolerance must be positive");
    require(op.size() < 0 || n == op.size(), "cg: operator must be square and match b");
    const int jacobi = cfg.jacobi ? 1 : 0;
    if (jacobi) require(diag != nullptr, "cg: jacobi preconditioner needs the diagonal");
    require(cfg.max_iterations >= 0, "cg: max_iterations must be >= 0");

    DevBuf<double> r(n), p(n), q(n), hist(cfg.max_iterations + 1);
    // CG reductions use 2 x kRedGridMax partials; the SpMV-fused p.q a
    // two-level grid sum over one CTA per 256 rows
    const int64_t spmv_blocks = (n + 255) / 256;
    const size_t npart = std::max<size_t>(2 * cg::kRedGridMax, cg::grid_sum_partials(spmv_blocks));
    DevBuf<double> partials(npart);
    DevBuf<unsigned> tickets(std::max<size_t>(1, cg::grid_sum_tickets(spmv_blocks)));
    EW_CUDA_CHECK(cudaMemsetAsync(tickets.get(), 0, tickets.bytes(), s));
    DevBuf<State> st(1);
    EW_CUDA_CHECK(cudaMemsetAsync(st.get(), 0, sizeof(State), s));
    if (n) EW_CUDA_CHECK(cudaMemsetAsync(x, 0, n * sizeof(double), s));
    const unsigned g = cg::red_grid(n);
    const unsigned gs = cg::resident_grid(cg::p_kernel, 256, n);
    const unsigned g_pq = cg::resident_grid(cg::pq_kernel<false>, cg::kRedBlock, n);
    const unsigned g_up = cg::resident_grid(cg::update_kernel<false>, cg::kRedBlock, n);

    cg::init_kernel<false><<<g, cg::kRedBlock, 0, s>>>(b, diag, n, jacobi, partials.get(), st.get());
    launched("cg::init_kernel");
    State h{};
    EW_CUDA_CHECK(cudaMemcpyAsync(&h, st.get(), sizeof(State), cudaMemcpyDeviceToHost, s));
    EW_CUDA_CHECK(cudaStreamSynchronize(s));
    if (h.status == cg::kBadRhs) throw Error(EW_CG_DIVERGENCE, "cg: non-finite right-hand side");
    require(!(h.flags & 2), "cg: zero diagonal entry under jacobi");
    if (h.bnorm == 0.0) {  // cg.cpp:45-49
        out.res.converged = 1;
        out.res.history_len = 1;
        out.history.assign(1, 0.0);
        return out;
    }

    // initial residual: one operator application on x0 = 0 (cg.cpp:52-57)
    op.apply(x, q.get(), s, nullptr);
    cg::start_kernel<false><<<g, cg::kRedBlock, 0, s>>>(b, diag, q.get(), r.get(), p.get(), n, jacobi,
                                                        cfg.rel_tolerance, partials.get(), st.get(), hist.get());
    launched("cg::start_kernel");

    State* hst = nullptr;
    EW_CUDA_CHECK(cudaMallocHost(&hst, 2 * sizeof(State)));
    cudaEvent_t ev[2] = {nullptr, nullptr};
    auto cleanup = [&] {
        if (ev[0]) cudaEventDestroy(ev[0]);
        if (ev[1]) cudaEventDestroy(ev[1]);
        cudaFreeHost(hst);
    };
    try {
        EW_CUDA_CHECK(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
        EW_CUDA_CHECK(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
        const int* done = &st.get()->done;
        const int64_t interval = cfg.recompute_interval;
        const bool host_op = op.host_callback();
        // a host closure cannot see the device flag: poll it before each call
        auto host_done = [&] {
            int d = 0;
            EW_CUDA_CHECK(cudaMemcpyAsync(&d, done, sizeof(int), cudaMemcpyDeviceToHost, s));
            EW_CUDA_CHECK(cudaStreamSynchronize(s));
            return d != 0;
        };
        int64_t it = 1;
        int batch = host_op ? 1 : 8, j = 0;
        bool stop = false;
        while (it <= cfg.max_iterations && !stop) {
            const int64_t last = std::min<int64_t>(cfg.max_iterations, it + batch - 1);
            for (; it <= last; ++it) {
                if (host_op && host_done()) {
                    stop = true;
                    break;
                }
                if (!op.apply_dot(p.get(), q.get(), s, done, DotSink{partials.get(), static_cast<unsigned>(npart), tickets.get(), st.get(), 0})) {
                    op.apply(p.get(), q.get(), s, done);
                    launch_pdl(cg::pq_kernel<false>, g_pq, cg::kRedBlock, s, p.get(), q.get(), n, partials.get(),
                               st.get());
                    launched("cg::pq_kernel");
                }
                const bool refresh = interval > 0 && it % interval == 0;
                launch_pdl(cg::update_kernel<false>, g_up, cg::kRedBlock, s, refresh ? 1 : 0, x, r.get(), p.get(),
                           q.get(), b, diag, n, jacobi, (long long)it, cfg.rel_tolerance, cfg.divergence_limit,
                           partials.get(), st.get(), hist.get());
                launched("cg::update_kernel");
                if (refresh) {
                    if (!(host_op && host_done())) op.apply(x, q.get(), s, done);
                    launch_pdl(cg::update_kernel<false>, g_up, cg::kRedBlock, s, 2, x, r.get(), p.get(), q.get(), b,
                               diag, n, jacobi, (long long)it, cfg.rel_tolerance, cfg.divergence_limit,
                               partials.get(), st.get(), hist.get());
                    launched("cg::update_kernel");
                }
                launch_pdl(cg::p_kernel, gs, 256, s, p.get(), r.get(), diag, n, jacobi, (const cg::State*)st.get());
                launched("cg::p_kernel");
            }
            // poll the previous batch's state while this batch runs
            const int slot = j & 1;
            EW_CUDA_CHECK(cudaMemcpyAsync(&hst[slot], st.get(), sizeof(State), cudaMemcpyDeviceToHost, s));
            EW_CUDA_CHECK(cudaEventRecord(ev[slot], s));
            if (j > 0) {
                EW_CUDA_CHECK(cudaEventSynchronize(ev[slot ^ 1]));
                if (hst[slot ^ 1].done) break;
            }
            ++j;
            if (!host_op) batch = std::min(batch * 2, 64);
        }
        EW_CUDA_CHECK(cudaMemcpyAsync(&hst[0], st.get(), sizeof(State), cudaMemcpyDeviceToHost, s));
        EW_CUDA_CHECK(cudaStreamSynchronize(s));
        h = hst[0];
    } catch (...) {
        cleanup();
        throw;
    }
    cleanup();
    return cg_outputs(h.status, h.iterations, cfg, hist.get());
}

CgOutputs cg_outputs(int status, long long iterations, const ew_cg_config& cfg, const double* hist_dev) {
    switch (status) {
        case cg::kBreakdown: throw Error(EW_CG_DIVERGENCE, "cg: breakdown, operator not positive definite");
        case cg::kNonFinite: throw Error(EW_CG_DIVERGENCE, "cg: non-finite residual");
        case cg::kDiverged: throw Error(EW_CG_DIVERGENCE, "cg: residual diverged");
        default: break;
    }
    CgOutputs out;
    out.res.iterations = iterations;
    out.res.converged = status == cg::kConverged ? 1 : 0;
    // one SpMV for x0, one per iteration, one per refresh (test_solver.cpp:55)
    out.res.spmv_calls =
        1 + iterations + (cfg.recompute_interval > 0 ? iterations / cfg.recompute_interval : 0);
    out.res.history_len = iterations + 1;
    out.history.resize(static_cast<size_t>(out.res.history_len));
    EW_CUDA_CHECK(cudaMemcpy(out.history.data(), hist_dev, out.history.size() * sizeof(double),
                             cudaMemcpyDeviceToHost));
    return out;
}

}  // namespace ew

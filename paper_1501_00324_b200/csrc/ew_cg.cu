// Single-GPU Jacobi PCG driver (cg.cpp:25-104): the prepared kernel (or a
// host closure) is the operator, everything else stays on the device.
//
// Per iteration, stream-ordered, no host round trip:
//   1. q = A p, with one p.q partial per SpMV CTA   (operator)
//   2. p.q summed in a fixed order                  (+ breakdown test, alpha)
//   3. x += alpha p ; r -= alpha q                  (+ r.r, r.z with z = r / diag,
//                                                    history, convergence /
//                                                    divergence, beta)
//      refresh iterations (k % recompute_interval == 0) replace the r update
//      by r = b - A x after one more operator launch, as cg.cpp:82-86
//   4. p = z + beta p
// Element-wise arithmetic follows the reference exactly; dot products are
// fixed-order trees (ew_cg.cuh). The iteration counter and a `done` flag live
// on the device, so one refresh interval of iterations is captured once into
// a CUDA graph and replayed; the host polls the state once per replay. The
// working set (vectors, partials, polling slots, graph) stays with the
// prepared kernel between solves.
#include "ew_cg.cuh"

namespace ew {

using cg::State;

namespace {

// One solve on working set w (sized and, for a device operator, holding the
// captured graph of one block of iterations).
CgOutputs cg_run(const CgOperator& op, CgWorkspace& w, const double* b_in, const double* diag_in, int64_t n,
                 const ew_cg_config& cfg, double* x_out, cudaStream_t s) {
    CgOutputs out;
    const int jacobi = cfg.jacobi ? 1 : 0;
    // CG reductions use 2 x kRedGridMax partials; the SpMV-fused p.q one per
    // SpMV CTA plus its final two-level sum
    const int64_t spmv_blocks = (std::max<int64_t>(n, op.spmv_threads()) + 255) / 256;
    const size_t npart = std::max<size_t>(2 * cg::kRedGridMax, cg::dot_partials(spmv_blocks));
    if (w.n != n || w.partials.size() < npart) {
        w.r.alloc(n), w.p.alloc(n), w.q.alloc(n), w.x.alloc(n), w.b.alloc(n), w.diag.alloc(n);
        w.partials.alloc(npart);
        w.tickets.alloc(std::max<size_t>(1, cg::dot_tickets(spmv_blocks)));
        w.st.alloc(1);
        w.n = n;
        if (w.exec) cudaGraphExecDestroy(w.exec);
        w.exec = nullptr;
    }
    if (static_cast<int64_t>(w.hist.size()) < cfg.max_iterations + 1) {
        w.hist.alloc(cfg.max_iterations + 1);
        if (w.exec) cudaGraphExecDestroy(w.exec);
        w.exec = nullptr;
    }
    if (!w.hst) EW_CUDA_CHECK(cudaMallocHost(&w.hst, 2 * sizeof(State)));
    for (auto& e : w.ev)
        if (!e) EW_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    State* hst = static_cast<State*>(w.hst);
    double *r = w.r.get(), *p = w.p.get(), *q = w.q.get(), *x = w.x.get(), *b = w.b.get(), *hist = w.hist.get();
    const double* diag = jacobi ? w.diag.get() : nullptr;
    State* st = w.st.get();
    double* partials = w.partials.get();

    // inputs into the working set, so a captured graph sees the same pointers
    if (n) {
        EW_CUDA_CHECK(cudaMemcpyAsync(b, b_in, n * 8, cudaMemcpyDeviceToDevice, s));
        if (jacobi) EW_CUDA_CHECK(cudaMemcpyAsync(w.diag.get(), diag_in, n * 8, cudaMemcpyDeviceToDevice, s));
        EW_CUDA_CHECK(cudaMemsetAsync(x, 0, n * sizeof(double), s));
    }
    EW_CUDA_CHECK(cudaMemsetAsync(w.tickets.get(), 0, w.tickets.bytes(), s));
    EW_CUDA_CHECK(cudaMemsetAsync(st, 0, sizeof(State), s));
    const long long max_it = cfg.max_iterations;
    EW_CUDA_CHECK(cudaMemcpyAsync(&st->max_it, &max_it, sizeof(max_it), cudaMemcpyHostToDevice, s));
    const unsigned g = cg::red_grid(n);
    const unsigned gs = cg::resident_grid(cg::p_kernel, 256, n);
    const unsigned g_pq = cg::resident_grid(cg::pq_kernel<false>, cg::kRedBlock, n);
    const unsigned g_up = cg::resident_grid(cg::update_kernel<false>, cg::kRedBlock, n);

    cg::init_kernel<false><<<g, cg::kRedBlock, 0, s>>>(b, diag, n, jacobi, partials, st);
    launched("cg::init_kernel");
    EW_CUDA_CHECK(cudaMemcpyAsync(&hst[0], st, sizeof(State), cudaMemcpyDeviceToHost, s));
    EW_CUDA_CHECK(cudaStreamSynchronize(s));
    if (hst[0].status == cg::kBadRhs) throw Error(EW_CG_DIVERGENCE, "cg: non-finite right-hand side");
    require(!(hst[0].flags & 2), "cg: zero diagonal entry under jacobi");
    if (hst[0].bnorm == 0.0) {  // cg.cpp:45-49
        out.res.converged = 1;
        out.res.history_len = 1;
        out.history.assign(1, 0.0);
        if (n) EW_CUDA_CHECK(cudaMemcpyAsync(x_out, x, n * 8, cudaMemcpyDeviceToDevice, s));
        EW_CUDA_CHECK(cudaStreamSynchronize(s));
        return out;
    }

    // initial residual: one operator application on x0 = 0 (cg.cpp:52-57)
    op.apply(x, q, s, nullptr);
    cg::start_kernel<false><<<g, cg::kRedBlock, 0, s>>>(b, diag, q, r, p, n, jacobi, cfg.rel_tolerance, partials, st,
                                                        hist);
    launched("cg::start_kernel");

    const int* done = &st->done;
    const int64_t interval = cfg.recompute_interval;
    const bool host_op = op.host_callback();
    // a host closure cannot see the device flag: poll it before each call
    auto host_done = [&] {
        int d = 0;
        EW_CUDA_CHECK(cudaMemcpyAsync(&d, done, sizeof(int), cudaMemcpyDeviceToHost, s));
        EW_CUDA_CHECK(cudaStreamSynchronize(s));
        return d != 0;
    };
    // one iteration k (cg.cpp:69-101) on stream t; k only selects the launch
    // pattern (refresh); the kernels count iterations on the device
    auto iteration = [&](int64_t k, cudaStream_t t) {
        if (!op.apply_dot(p, q, t, done,
                          DotSink{partials, static_cast<unsigned>(npart), w.tickets.get(), st, 0})) {
            op.apply(p, q, t, done);
            launch_pdl(cg::pq_kernel<false>, g_pq, cg::kRedBlock, t, (const double*)p, (const double*)q, n, partials,
                       st);
            launched("cg::pq_kernel");
        }
        const bool refresh = interval > 0 && k % interval == 0;
        launch_pdl(cg::update_kernel<false>, g_up, cg::kRedBlock, t, refresh ? 1 : 0, x, r, (const double*)p,
                   (const double*)q, (const double*)b, diag, n, jacobi, cfg.rel_tolerance,
                   cfg.divergence_limit, partials, st, hist);
        launched("cg::update_kernel");
        if (refresh) {
            if (!(host_op && host_done())) op.apply(x, q, t, done);
            launch_pdl(cg::update_kernel<false>, g_up, cg::kRedBlock, t, 2, x, r, (const double*)p, (const double*)q,
                       (const double*)b, diag, n, jacobi, cfg.rel_tolerance, cfg.divergence_limit,
                       partials, st, hist);
            launched("cg::update_kernel");
        }
        launch_pdl(cg::p_kernel, gs, 256, t, p, (const double*)r, diag, n, jacobi, (const cg::State*)st);
        launched("cg::p_kernel");
    };
    // the state of the previous block is polled while this block runs
    int j = 0;
    auto poll = [&]() -> bool {
        const int slot = j & 1;
        EW_CUDA_CHECK(cudaMemcpyAsync(&hst[slot], st, sizeof(State), cudaMemcpyDeviceToHost, s));
        EW_CUDA_CHECK(cudaEventRecord(w.ev[slot], s));
        bool stop = false;
        if (j > 0) {
            EW_CUDA_CHECK(cudaEventSynchronize(w.ev[slot ^ 1]));
            stop = hst[slot ^ 1].done != 0;
        }
        ++j;
        return stop;
    };
    if (host_op) {
        for (int64_t it = 1; it <= cfg.max_iterations; ++it) {
            if (host_done()) break;
            iteration(it, s);
        }
    } else if (cfg.max_iterations > 0) {
        // Device operator: one CUDA graph of a block of B iterations (one
        // refresh interval, the refresh iteration last), replayed; the device
        // iteration counter and `done` flag make the iterations past
        // convergence or max_iterations no-ops. Captured once per working set
        // and configuration.
        const int64_t B = interval > 0 ? interval : 32;
        const bool same = w.exec && w.g_tol == cfg.rel_tolerance && w.g_div == cfg.divergence_limit &&
                          w.g_interval == interval && w.g_jacobi == jacobi &&
                          w.g_hist == static_cast<int64_t>(w.hist.size());
        if (!same) {
            if (w.exec) cudaGraphExecDestroy(w.exec);
            w.exec = nullptr;
            if (!w.cap) EW_CUDA_CHECK(cudaStreamCreateWithFlags(&w.cap, cudaStreamNonBlocking));
            const int64_t before = g_launches.load();
            cudaGraph_t graph = nullptr;
            EW_CUDA_CHECK(cudaStreamBeginCapture(w.cap, cudaStreamCaptureModeThreadLocal));
            try {
                for (int64_t k = 1; k <= B; ++k) iteration(k, w.cap);
            } catch (...) {
                cudaStreamEndCapture(w.cap, &graph);
                if (graph) cudaGraphDestroy(graph);
                throw;
            }
            EW_CUDA_CHECK(cudaStreamEndCapture(w.cap, &graph));
            const cudaError_t e = cudaGraphInstantiate(&w.exec, graph, 0);
            cudaGraphDestroy(graph);
            EW_CUDA_CHECK(e);
            w.per_block = g_launches.load() - before;
            g_launches.fetch_sub(w.per_block, std::memory_order_relaxed);  // counted per replay below
            w.g_tol = cfg.rel_tolerance, w.g_div = cfg.divergence_limit, w.g_interval = interval;
            w.g_jacobi = jacobi, w.g_hist = static_cast<int64_t>(w.hist.size());
        }
        const int64_t blocks = (cfg.max_iterations + B - 1) / B;
        for (int64_t blk = 0; blk < blocks; ++blk) {
            EW_CUDA_CHECK(cudaGraphLaunch(w.exec, s));
            g_launches.fetch_add(w.per_block, std::memory_order_relaxed);
            if (poll()) break;
        }
    }
    EW_CUDA_CHECK(cudaMemcpyAsync(&hst[0], st, sizeof(State), cudaMemcpyDeviceToHost, s));
    if (n) EW_CUDA_CHECK(cudaMemcpyAsync(x_out, x, n * 8, cudaMemcpyDeviceToDevice, s));
    EW_CUDA_CHECK(cudaStreamSynchronize(s));
    return cg_outputs(hst[0].status, hst[0].iterations, cfg, hist);
}

}  // namespace

CgOutputs cg_device(const CgOperator& op, const double* b, const double* diag, int64_t n,
                    const ew_cg_config& cfg, double* x, cudaStream_t s) {
    require(cfg.rel_tolerance > 0.0, "cg: tolerance must be positive");
    require(op.size() < 0 || n == op.size(), "cg: operator must be square and match b");
    if (cfg.jacobi) require(diag != nullptr, "cg: jacobi preconditioner needs the diagonal");
    require(cfg.max_iterations >= 0, "cg: max_iterations must be >= 0");
    if (CgWorkspace* w = op.workspace()) {
        std::unique_lock<std::mutex> lock(w->mu, std::try_to_lock);
        if (lock.owns_lock()) return cg_run(op, *w, b, diag, n, cfg, x, s);
    }
    CgWorkspace tmp;  // a host closure, or a concurrent solve on the same kernel
    return cg_run(op, tmp, b, diag, n, cfg, x, s);
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

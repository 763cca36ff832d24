// Jacobi-preconditioned CG on the device (cg.cpp:25-104), driving a prepared
// ELL-WARP kernel as its operator.
//
// Each iteration is four stream-ordered launches with no host round trip:
//   1. q = A p                      (the kernel's operator)
//   2. pq = p.q                     (+ breakdown test, alpha = rz / pq)
//   3. x += alpha p ; r -= alpha q  (+ r.r, r.z with z = r / diag, the
//                                    residual history entry, convergence /
//                                    divergence tests, beta = rz' / rz)
//      on refresh iterations (k % recompute_interval == 0) the r update is
//      replaced by r = b - A x after one more operator launch, as cg.cpp:78-81
//   4. p = z + beta p
// The element-wise arithmetic follows the reference exactly (separately
// rounded mul / add / div); only the dot products differ in summation order
// (fixed-shape, deterministic two-level trees instead of a sequential sum),
// which the parity tests bound with the reference's own comparator
// |dh| <= 1e-10 (1 + h) (test_solver.cpp:109-110).
//
// Every kernel reads a device `done` flag first, so the host enqueues
// iterations in batches and only polls the flag once per batch.
#include <cmath>

#include "ew_internal.cuh"

namespace ew {

namespace {

enum CgStatus : int {
    kRunning = 0,
    kConverged = 1,
    kBreakdown = 2,
    kNonFinite = 3,
    kDiverged = 4,
    kBadRhs = 5,
    kZeroDiag = 6,
};

struct CgState {
    double rz, pq, alpha, beta, bnorm, rr, rz_new;
    int done, status;
    long long iterations;
    unsigned int ticket;  // last-block election counter
    int nonfinite;        // any non-finite residual entry this iteration
};

constexpr int kRedBlock = 256;
constexpr int kRedGridMax = 148 * 4;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, o));
    return v;
}

// Deterministic block sum of NV values; result valid in thread 0.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV]) {
    __shared__ double sh[NV][kRedBlock / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        v[i] = warp_sum(v[i]);
        if (lane == 0) sh[i][wid] = v[i];
    }
    __syncthreads();
    if (wid == 0) {
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            double t = lane < kRedBlock / 32 ? sh[i][lane] : 0.0;
            v[i] = warp_sum(t);
        }
    }
}

// Writes this block's partials; returns true in thread 0 of the last block to
// finish, after which `partials` holds every block's sums (fixed order).
template <int NV>
__device__ __forceinline__ bool publish_partials(double (&v)[NV], double* partials,
                                                 unsigned int* ticket) {
    __shared__ bool last;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < NV; ++i) partials[i * gridDim.x + blockIdx.x] = v[i];
        __threadfence();
        const unsigned int t = atomicAdd(ticket, 1u);
        last = (t == gridDim.x - 1);
    }
    __syncthreads();
    return last;
}

// Sum of the grid's partials by the last block, in a fixed order.
template <int NV>
__device__ __forceinline__ void final_sum(double (&out)[NV], const double* partials) {
    double v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        double t = 0.0;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
            t = __dadd_rn(t, *((volatile const double*)&partials[i * gridDim.x + b]));
        v[i] = t;
    }
    block_sum<NV>(v);
#pragma unroll
    for (int i = 0; i < NV; ++i) out[i] = v[i];
}

// Pre-checks of cg.cpp:28-33 and ||b|| (cg.cpp:44).
__global__ void cg_init_kernel(const double* __restrict__ b, const double* __restrict__ diag,
                               int64_t n, int jacobi, double* partials, CgState* st) {
    double v[1] = {0.0};
    int bad_b = 0, zero_d = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double bi = b[i];
        if (!isfinite(bi)) bad_b = 1;
        if (jacobi && diag[i] == 0.0) zero_d = 1;
        v[0] = __dadd_rn(v[0], __dmul_rn(bi, bi));
    }
    if (bad_b) atomicMax(&st->status, (int)kBadRhs);
    if (zero_d) atomicOr(&st->nonfinite, 2);
    block_sum<1>(v);
    if (!publish_partials<1>(v, partials, &st->ticket)) return;
    double tot[1];
    final_sum<1>(tot, partials);
    if (threadIdx.x == 0) {
        st->ticket = 0;
        st->bnorm = sqrt(tot[0]);
    }
}

// r = b - A x0, history[0], z = r / diag, p = z, rz = r.z (cg.cpp:50-66)
__global__ void cg_start_kernel(const double* __restrict__ b, const double* __restrict__ diag,
                                const double* __restrict__ ax, double* __restrict__ r,
                                double* __restrict__ p, int64_t n, int jacobi, double tol,
                                double* partials, CgState* st, double* hist) {
    double v[2] = {0.0, 0.0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double ri = __dsub_rn(b[i], ax[i]);
        r[i] = ri;
        const double zi = jacobi ? __ddiv_rn(ri, diag[i]) : ri;
        p[i] = zi;
        v[0] = __dadd_rn(v[0], __dmul_rn(ri, ri));
        v[1] = __dadd_rn(v[1], __dmul_rn(ri, zi));
    }
    block_sum<2>(v);
    if (!publish_partials<2>(v, partials, &st->ticket)) return;
    double tot[2];
    final_sum<2>(tot, partials);
    if (threadIdx.x == 0) {
        st->ticket = 0;
        const double rel = sqrt(tot[0]) / st->bnorm;
        hist[0] = rel;
        st->rz = tot[1];
        st->iterations = 0;
        if (rel <= tol) {
            st->status = kConverged;
            st->done = 1;
        }
    }
}

// pq = p.q; breakdown unless finite and > 0 (cg.cpp:72-77); alpha = rz / pq.
__global__ void cg_pq_kernel(const double* __restrict__ p, const double* __restrict__ q, int64_t n,
                             double* partials, CgState* st) {
    if (st->done) return;
    double v[1] = {0.0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        v[0] = __dadd_rn(v[0], __dmul_rn(p[i], q[i]));
    block_sum<1>(v);
    if (!publish_partials<1>(v, partials, &st->ticket)) return;
    double tot[1];
    final_sum<1>(tot, partials);
    if (threadIdx.x == 0) {
        st->ticket = 0;
        const double pq = tot[0];
        st->pq = pq;
        if (!isfinite(pq) || pq <= 0.0) {
            st->status = kBreakdown;
            st->done = 1;
        } else {
            st->alpha = st->rz / pq;
        }
    }
}

// Residual bookkeeping shared by the update kernels (cg.cpp:82-101), run by
// thread 0 of the last block with the grid totals rr = r.r, rz' = r.z.
__device__ __forceinline__ void cg_finish_iteration(CgState* st, double rr, double rz_new,
                                                    long long k, double tol, double divergence,
                                                    double* hist) {
    if (st->nonfinite & 1) {  // check_finite(r) (cg.cpp:87)
        st->status = kNonFinite;
        st->done = 1;
        return;
    }
    st->iterations = k;
    const double rel = sqrt(rr) / st->bnorm;
    hist[k] = rel;
    if (rel > divergence) {
        st->status = kDiverged;
        st->done = 1;
        return;
    }
    if (rel <= tol) {
        st->status = kConverged;
        st->done = 1;
        return;
    }
    st->beta = rz_new / st->rz;
    st->rz = rz_new;
}

// mode 0: x += alpha p, r -= alpha q, then the residual bookkeeping.
// mode 1 (refresh, first half): x += alpha p only.
// mode 2 (refresh, second half): r = b - A x (ax in q), then bookkeeping.
__global__ void cg_update_kernel(int mode, double* __restrict__ x, double* __restrict__ r,
                                 const double* __restrict__ p, const double* __restrict__ q,
                                 const double* __restrict__ b, const double* __restrict__ diag,
                                 int64_t n, int jacobi, long long k, double tol, double divergence,
                                 double* partials, CgState* st, double* hist) {
    if (st->done) return;
    const double alpha = st->alpha;
    double v[2] = {0.0, 0.0};
    int bad = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double ri;
        if (mode != 2) x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
        if (mode == 1) continue;
        if (mode == 0) {
            ri = __dsub_rn(r[i], __dmul_rn(alpha, q[i]));
        } else {
            ri = __dsub_rn(b[i], q[i]);
        }
        r[i] = ri;
        if (!isfinite(ri)) bad = 1;
        const double zi = jacobi ? __ddiv_rn(ri, diag[i]) : ri;
        v[0] = __dadd_rn(v[0], __dmul_rn(ri, ri));
        v[1] = __dadd_rn(v[1], __dmul_rn(ri, zi));
    }
    if (mode == 1) return;
    if (bad) atomicOr(&st->nonfinite, 1);
    block_sum<2>(v);
    if (!publish_partials<2>(v, partials, &st->ticket)) return;
    double tot[2];
    final_sum<2>(tot, partials);
    if (threadIdx.x == 0) {
        st->ticket = 0;
        st->rr = tot[0];
        st->rz_new = tot[1];
        cg_finish_iteration(st, tot[0], tot[1], k, tol, divergence, hist);
    }
}

// p = z + beta p (cg.cpp:96-99)
__global__ void cg_p_kernel(double* __restrict__ p, const double* __restrict__ r,
                            const double* __restrict__ diag, int64_t n, int jacobi,
                            const CgState* st) {
    if (st->done) return;
    const double beta = st->beta;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double zi = jacobi ? __ddiv_rn(r[i], diag[i]) : r[i];
        p[i] = __dadd_rn(zi, __dmul_rn(beta, p[i]));
    }
}

unsigned red_grid(int64_t n) {
    int64_t g = (n + kRedBlock - 1) / kRedBlock;
    if (g > kRedGridMax) g = kRedGridMax;
    return static_cast<unsigned>(g < 1 ? 1 : g);
}

unsigned stream_grid(int64_t n) {
    int64_t g = (n + kBlock - 1) / kBlock;
    if (g > 148 * 16) g = 148 * 16;
    return static_cast<unsigned>(g < 1 ? 1 : g);
}

}  // namespace

CgOutputs cg_device(const CgOperator& op, const double* b, const double* diag, int64_t n,
                    const ew_cg_config& cfg, double* x, cudaStream_t s) {
    CgOutputs out;
    require(cfg.rel_tolerance > 0.0, "cg: tolerance must be positive");
    require(op.size() < 0 || n == op.size(), "cg: operator must be square and match b");
    const int jacobi = cfg.jacobi ? 1 : 0;
    if (jacobi) require(diag != nullptr, "cg: jacobi preconditioner needs the diagonal");
    require(cfg.max_iterations >= 0, "cg: max_iterations must be >= 0");

    DevBuf<double> r(n), p(n), q(n), hist(cfg.max_iterations + 1);
    DevBuf<double> partials(2 * kRedGridMax);
    DevBuf<CgState> st(1);
    EW_CUDA_CHECK(cudaMemsetAsync(st.get(), 0, sizeof(CgState), s));
    if (n) EW_CUDA_CHECK(cudaMemsetAsync(x, 0, n * sizeof(double), s));
    const unsigned g = red_grid(n);
    const unsigned gs = stream_grid(n);

    cg_init_kernel<<<g, kRedBlock, 0, s>>>(b, diag, n, jacobi, partials.get(), st.get());
    launched("cg_init_kernel");
    CgState h{};
    EW_CUDA_CHECK(cudaMemcpyAsync(&h, st.get(), sizeof(CgState), cudaMemcpyDeviceToHost, s));
    EW_CUDA_CHECK(cudaStreamSynchronize(s));
    if (h.status == kBadRhs) throw Error(EW_CG_DIVERGENCE, "cg: non-finite right-hand side");
    require(!(h.nonfinite & 2), "cg: zero diagonal entry under jacobi");
    if (h.bnorm == 0.0) {  // cg.cpp:45-49
        out.res.converged = 1;
        out.res.iterations = 0;
        out.res.spmv_calls = 0;
        out.res.history_len = 1;
        out.history.assign(1, 0.0);
        return out;
    }

    // initial residual: one operator application on x0 = 0 (cg.cpp:52-57)
    op.apply(x, q.get(), s, nullptr);
    cg_start_kernel<<<g, kRedBlock, 0, s>>>(b, diag, q.get(), r.get(), p.get(), n, jacobi,
                                            cfg.rel_tolerance, partials.get(), st.get(), hist.get());
    launched("cg_start_kernel");

    CgState* hst = nullptr;
    EW_CUDA_CHECK(cudaMallocHost(&hst, 2 * sizeof(CgState)));
    cudaEvent_t ev[2];
    EW_CUDA_CHECK(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
    EW_CUDA_CHECK(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
    auto cleanup = [&] {
        cudaEventDestroy(ev[0]);
        cudaEventDestroy(ev[1]);
        cudaFreeHost(hst);
    };
    try {
        int64_t it = 1;
        int batch = 8, j = 0;
        bool stop = false;
        const int* done = &st.get()->done;
        const int64_t interval = cfg.recompute_interval;
        const bool host_op = op.host_callback();
        // a host closure cannot see the device flag: poll it before each call
        auto host_done = [&] {
            int h_done = 0;
            EW_CUDA_CHECK(cudaMemcpyAsync(&h_done, done, sizeof(int), cudaMemcpyDeviceToHost, s));
            EW_CUDA_CHECK(cudaStreamSynchronize(s));
            return h_done != 0;
        };
        if (host_op) batch = 1;
        while (it <= cfg.max_iterations && !stop) {
            const int64_t last = std::min<int64_t>(cfg.max_iterations, it + batch - 1);
            for (; it <= last; ++it) {
                if (host_op && host_done()) {
                    stop = true;
                    break;
                }
                op.apply(p.get(), q.get(), s, done);
                cg_pq_kernel<<<g, kRedBlock, 0, s>>>(p.get(), q.get(), n, partials.get(), st.get());
                launched("cg_pq_kernel");
                const bool refresh = interval > 0 && it % interval == 0;
                if (!refresh) {
                    cg_update_kernel<<<g, kRedBlock, 0, s>>>(0, x, r.get(), p.get(), q.get(), b, diag, n,
                                                             jacobi, it, cfg.rel_tolerance,
                                                             cfg.divergence_limit, partials.get(),
                                                             st.get(), hist.get());
                    launched("cg_update_kernel");
                } else {
                    cg_update_kernel<<<g, kRedBlock, 0, s>>>(1, x, r.get(), p.get(), q.get(), b, diag, n,
                                                             jacobi, it, cfg.rel_tolerance,
                                                             cfg.divergence_limit, partials.get(),
                                                             st.get(), hist.get());
                    launched("cg_update_kernel");
                    if (!(host_op && host_done())) op.apply(x, q.get(), s, done);
                    cg_update_kernel<<<g, kRedBlock, 0, s>>>(2, x, r.get(), p.get(), q.get(), b, diag, n,
                                                             jacobi, it, cfg.rel_tolerance,
                                                             cfg.divergence_limit, partials.get(),
                                                             st.get(), hist.get());
                    launched("cg_update_kernel");
                }
                cg_p_kernel<<<gs, kBlock, 0, s>>>(p.get(), r.get(), diag, n, jacobi, st.get());
                launched("cg_p_kernel");
            }
            // poll the previous batch's state while this batch runs
            const int slot = j & 1;
            EW_CUDA_CHECK(cudaMemcpyAsync(&hst[slot], st.get(), sizeof(CgState), cudaMemcpyDeviceToHost, s));
            EW_CUDA_CHECK(cudaEventRecord(ev[slot], s));
            if (j > 0) {
                EW_CUDA_CHECK(cudaEventSynchronize(ev[slot ^ 1]));
                if (hst[slot ^ 1].done) break;
            }
            ++j;
            if (!host_op) batch = std::min(batch * 2, 64);
        }
        EW_CUDA_CHECK(cudaMemcpyAsync(&hst[0], st.get(), sizeof(CgState), cudaMemcpyDeviceToHost, s));
        EW_CUDA_CHECK(cudaStreamSynchronize(s));
        h = hst[0];
    } catch (...) {
        cleanup();
        throw;
    }
    cleanup();

    switch (h.status) {
        case kBreakdown:
            throw Error(EW_CG_DIVERGENCE, "cg: breakdown, operator not positive definite");
        case kNonFinite:
            throw Error(EW_CG_DIVERGENCE, "cg: non-finite residual");
        case kDiverged:
            throw Error(EW_CG_DIVERGENCE, "cg: residual diverged");
        default:
            break;
    }
    out.res.iterations = h.iterations;
    out.res.converged = h.status == kConverged ? 1 : 0;
    out.res.spmv_calls = 1 + h.iterations +
                         (cfg.recompute_interval > 0 ? h.iterations / cfg.recompute_interval : 0);
    out.res.history_len = h.iterations + 1;
    out.history.resize(static_cast<size_t>(out.res.history_len));
    EW_CUDA_CHECK(cudaMemcpy(out.history.data(), hist.get(), out.history.size() * sizeof(double),
                             cudaMemcpyDeviceToHost));
    return out;
}

}  // namespace ew

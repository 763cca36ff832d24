// Device kernels of the Jacobi PCG (cg.cpp:25-104), shared by the
// single-GPU solver (ew_cg.cu) and the row-partitioned one (ew_dist.cu).
//
// Every reduction is deterministic: each CTA sums a fixed grid-stride subset
// of the rows, CTA partials are combined by the last CTA to finish in CTA
// order. With DIST = false that last CTA also applies the reference's
// decision (alpha, breakdown, convergence, divergence, beta). With DIST =
// true it only stores this partition's totals in State::loc; the transport
// all-gathers them and cg_finalize_kernel sums the partitions in rank order
// and applies the same decision on every rank.
#pragma once

#include <cmath>

#include "ew_internal.cuh"

namespace ew {
namespace cg {

enum Status : int {
    kRunning = 0,
    kConverged = 1,
    kBreakdown = 2,
    kNonFinite = 3,
    kDiverged = 4,
    kBadRhs = 5,
};

enum What : int { kBnorm = 0, kStart = 1, kPq = 2, kUpdate = 3 };

struct State {
    double rz, pq, alpha, beta, bnorm, rr, rz_new;
    int done, status;
    long long iterations;
    long long cur_it;     // iteration the reductions belong to (advanced by decide_pq)
    long long max_it;     // CgConfig::max_iterations (set by the host before the solve)
    unsigned int ticket;  // last-CTA election counter
    int flags;            // bit 0: non-finite residual entry; bit 1: zero diagonal
    double loc[2];        // DIST: this partition's totals of the current reduction
};

constexpr int kRedBlock = 256;
constexpr int kRedGridMax = 148 * 8;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, o));
    return v;
}

// Deterministic CTA sum of NV values; result valid in thread 0.
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
        for (int i = 0; i < NV; ++i) v[i] = warp_sum(lane < kRedBlock / 32 ? sh[i][lane] : 0.0);
    }
}

// Publishes this CTA's sums; true in every thread of the last CTA to finish.
template <int NV>
__device__ __forceinline__ bool publish_partials(const double (&v)[NV], double* partials, unsigned int* ticket) {
    __shared__ bool last;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < NV; ++i) partials[i * gridDim.x + blockIdx.x] = v[i];
        __threadfence();
        last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    return last;
}

template <int NV>
__device__ __forceinline__ void final_sum(double (&out)[NV], const double* partials) {
    // Thread t sums partials t, t + blockDim, ... in that order; the loads
    // are issued together (L2, past L1) rather than one dependent load per
    // step. Grids are at most kRedGridMax CTAs.
    constexpr int kMaxPer = (kRedGridMax + kRedBlock - 1) / kRedBlock;
    double v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        double ld[kMaxPer];
#pragma unroll
        for (int u = 0; u < kMaxPer; ++u) {
            const int b = threadIdx.x + u * blockDim.x;
            ld[u] = b < (int)gridDim.x ? __ldcg(&partials[i * gridDim.x + b]) : 0.0;
        }
        double t = 0.0;
#pragma unroll
        for (int u = 0; u < kMaxPer; ++u)
            if (threadIdx.x + u * blockDim.x < gridDim.x) t = __dadd_rn(t, ld[u]);
        v[i] = t;
    }
    block_sum<NV>(v);
#pragma unroll
    for (int i = 0; i < NV; ++i) out[i] = v[i];
}

// Two-level deterministic grid sum for plain (one CTA per 256 rows) grids of
// any size, finished inside the kernel: every CTA publishes its sum; the
// last CTA of each group of kRedBlock CTAs sums the group in CTA order; the
// last group to finish sums the group totals in group order. The order of
// every addition is fixed by the grid shape alone. partials holds
// gridDim.x + ngroups doubles, tickets ngroups zeroed counters (left zeroed).
// True in thread 0 of the one CTA that holds the total.
__device__ __forceinline__ bool grid_sum(double v, double* partials, unsigned* tickets, unsigned* top,
                                         double& total) {
    __shared__ bool last;
    const unsigned G = gridDim.x, g = blockIdx.x / kRedBlock, ng = (G + kRedBlock - 1) / kRedBlock;
    const unsigned gsize = min(static_cast<unsigned>(kRedBlock), G - g * kRedBlock);
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = v;
        __threadfence();
        last = atomicAdd(&tickets[g], 1u) == gsize - 1;
    }
    __syncthreads();
    if (!last) return false;
    __threadfence();
    double t[1] = {threadIdx.x < gsize ? __ldcg(&partials[g * kRedBlock + threadIdx.x]) : 0.0};
    block_sum<1>(t);
    if (threadIdx.x == 0) {
        tickets[g] = 0;
        partials[G + g] = t[0];
        __threadfence();
        last = atomicAdd(top, 1u) == ng - 1;
    }
    __syncthreads();
    if (!last) return false;
    __threadfence();
    double u[1] = {0.0};
    for (unsigned i = threadIdx.x; i < ng; i += blockDim.x) u[0] = __dadd_rn(u[0], __ldcg(&partials[G + i]));
    block_sum<1>(u);
    if (threadIdx.x != 0) return false;
    *top = 0;
    total = u[0];
    return true;
}

// partials / tickets a plain grid of `nblocks` CTAs needs for grid_sum
inline size_t grid_sum_partials(int64_t nblocks) {
    return static_cast<size_t>(nblocks + (nblocks + kRedBlock - 1) / kRedBlock);
}
inline size_t grid_sum_tickets(int64_t nblocks) { return static_cast<size_t>((nblocks + kRedBlock - 1) / kRedBlock); }

// ---- decisions (cg.cpp), applied to global totals by one thread ----------
__device__ __forceinline__ void decide_bnorm(State* st, double bb) { st->bnorm = sqrt(bb); }

__device__ __forceinline__ void decide_start(State* st, double rr, double rz, double tol, double* hist) {
    const double rel = sqrt(rr) / st->bnorm;  // cg.cpp:58
    hist[0] = rel;
    st->rz = rz;
    st->iterations = 0;
    if (rel <= tol) {
        st->status = kConverged;
        st->done = 1;
    }
}

__device__ __forceinline__ void decide_pq(State* st, double pq) {
    // a new iteration; past max_iterations the loop has ended (cg.cpp:69),
    // not converged. Launches run ahead in whole blocks (CUDA graph) and
    // become no-ops from here on.
    const long long k = st->cur_it + 1;
    if (k > st->max_it) {
        st->done = 1;
        return;
    }
    st->cur_it = k;
    st->pq = pq;  // cg.cpp:72-77
    if (!isfinite(pq) || pq <= 0.0) {
        st->status = kBreakdown;
        st->done = 1;
    } else {
        st->alpha = st->rz / pq;
    }
}

__device__ __forceinline__ void decide_update(State* st, double rr, double rz_new, double tol, double divergence,
                                              double* hist) {
    const long long k = st->cur_it;
    st->rr = rr;
    st->rz_new = rz_new;
    // check_finite(r), cg.cpp:87. A non-finite entry makes r.r non-finite,
    // which is how the flag reaches every rank of a partitioned solve.
    if ((st->flags & 1) || !isfinite(rr)) {
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

// Ends a reduction kernel: last CTA either decides (single GPU) or stores
// the partition's totals (DIST).
template <bool DIST, int NV, typename Decide>
__device__ __forceinline__ void finish(const double (&v)[NV], double* partials, State* st, Decide&& decide) {
    double vv[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) vv[i] = v[i];
    block_sum<NV>(vv);
    if (!publish_partials<NV>(vv, partials, &st->ticket)) return;
    double tot[NV];
    final_sum<NV>(tot, partials);
    if (threadIdx.x == 0) {
        st->ticket = 0;
        if (DIST) {
#pragma unroll
            for (int i = 0; i < NV; ++i) st->loc[i] = tot[i];
            if (NV == 1) st->loc[1] = 0.0;  // p.q: the second row-set slot
        } else {
            decide(tot);
        }
    }
}

#define EW_GRID_STRIDE(i, n) \
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

// ||b||^2 and the pre-checks of cg.cpp:28-33
template <bool DIST>
__global__ void __launch_bounds__(kRedBlock) init_kernel(const double* __restrict__ b, const double* __restrict__ diag,
                                                         int64_t n, int jacobi, double* partials, State* st) {
    double v[1] = {0.0};
    int bad_b = 0, zero_d = 0;
    EW_GRID_STRIDE(i, n) {
        const double bi = b[i];
        bad_b |= !isfinite(bi);
        if (jacobi) zero_d |= diag[i] == 0.0;
        v[0] = __dadd_rn(v[0], __dmul_rn(bi, bi));
    }
    if (bad_b) atomicMax(&st->status, (int)kBadRhs);
    if (zero_d) atomicOr(&st->flags, 2);
    finish<DIST, 1>(v, partials, st, [&](const double (&t)[1]) { decide_bnorm(st, t[0]); });
}

// r = b - A x0, z = r / diag, p = z, r.r and r.z (cg.cpp:50-66)
template <bool DIST>
__global__ void __launch_bounds__(kRedBlock) start_kernel(const double* __restrict__ b, const double* __restrict__ diag,
                                                          const double* __restrict__ ax, double* __restrict__ r,
                                                          double* __restrict__ p, int64_t n, int jacobi, double tol,
                                                          double* partials, State* st, double* hist) {
    double v[2] = {0.0, 0.0};
    EW_GRID_STRIDE(i, n) {
        const double ri = __dsub_rn(b[i], ax[i]);
        r[i] = ri;
        const double zi = jacobi ? __ddiv_rn(ri, diag[i]) : ri;
        p[i] = zi;
        v[0] = __dadd_rn(v[0], __dmul_rn(ri, ri));
        v[1] = __dadd_rn(v[1], __dmul_rn(ri, zi));
    }
    finish<DIST, 2>(v, partials, st, [&](const double (&t)[2]) { decide_start(st, t[0], t[1], tol, hist); });
}

// The streaming kernels below take U elements per thread per round (indices
// i, i+S, ..., i+(U-1)S with S the grid's thread count) and issue every load
// of a round before the order-preserving arithmetic consumes them: U times
// the bytes in flight of a plain grid-stride loop, which alone is latency
// bound at the occupancy these kernels reach.
constexpr int kU = 4;
constexpr int kUpdU = 2;  // the update kernel's divisions cost registers: two per round
#define EW_ROUNDS_U(i0, S, n, U)                                                                 \
    for (int64_t S = (int64_t)gridDim.x * blockDim.x, i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; \
         i0 < (n); i0 += (U) * S)
#define EW_ROUNDS(i0, S, n) EW_ROUNDS_U(i0, S, n, kU)

// p.q (cg.cpp:72)
template <bool DIST>
__global__ void __launch_bounds__(kRedBlock) pq_kernel(const double* __restrict__ p, const double* __restrict__ q,
                                                       int64_t n, double* partials, State* st) {
    pdl_wait();
    if (st->done) return;
    double v[1] = {0.0};
    EW_ROUNDS(i0, S, n) {
        double a[kU], c[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int64_t i = i0 + u * S;
            a[u] = i < n ? p[i] : 0.0;
            c[u] = i < n ? q[i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kU; ++u)
            if (i0 + u * S < n) v[0] = __dadd_rn(v[0], __dmul_rn(a[u], c[u]));
    }
    pdl_trigger();
    finish<DIST, 1>(v, partials, st, [&](const double (&t)[1]) { decide_pq(st, t[0]); });
}

// L2 eviction hints for the vector kernels: data the next kernel reads again
// (r, diag, p: the p update) is kept, data it does not (x, q) goes first.
__device__ __forceinline__ uint64_t l2_policy_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t l2_policy_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ double ld_hint(const double* p, uint64_t pol) {
    double v;
    asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_hint(double* p, double v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}

// mode 0: x += alpha p, r -= alpha q, then r.r, r.z   (cg.cpp:78-81, 88-99)
// mode 1: x += alpha p only (refresh iteration, first half)
// mode 2: r = b - A x (A x in q), then r.r, r.z       (cg.cpp:82-86)
template <bool DIST>
__global__ void __launch_bounds__(kRedBlock, 4) update_kernel(int mode, double* __restrict__ x, double* __restrict__ r,
                                                           const double* __restrict__ p, const double* __restrict__ q,
                                                           const double* __restrict__ b,
                                                           const double* __restrict__ diag, int64_t n, int jacobi,
                                                           double tol, double divergence,
                                                           double* partials, State* st, double* hist) {
    const uint64_t first = l2_policy_first(), last = l2_policy_last();
    double xv[kUpdU], pv[kUpdU], qv[kUpdU], rv[kUpdU], dv[kUpdU];
    auto load = [&](int64_t i0, int64_t S) {
#pragma unroll
        for (int u = 0; u < kUpdU; ++u) {
            const int64_t i = i0 + u * S;
            const bool ok = i < n;
            xv[u] = ok && mode != 2 ? ld_hint(x + i, first) : 0.0;
            pv[u] = ok && mode != 2 ? ld_hint(p + i, last) : 0.0;
            qv[u] = ok && mode != 1 ? ld_hint(q + i, first) : 0.0;
            rv[u] = ok && mode != 1 ? (mode == 0 ? r[i] : b[i]) : 0.0;
            dv[u] = ok && mode != 1 && jacobi ? ld_hint(diag + i, last) : 1.0;
        }
    };
    // mode 0: the first round's loads go out before the wait for alpha and
    // overlap the p.q reduction's tail. Safe: x, p, r, diag are older, and q
    // comes from the SpMV, which the kernel before this one (dot_final or
    // pq_kernel, triggering only after its own wait; or a plain launch)
    // saw complete before this grid could start. Mode 2 reads a q that the
    // SpMV right before it is still writing: no early loads.
    const int64_t S0 = (int64_t)gridDim.x * blockDim.x, t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    bool have = mode == 0 && t0 < n;
    if (have) load(t0, S0);
    pdl_wait();
    if (st->done) return;
    const double alpha = st->alpha;
    double v[2] = {0.0, 0.0};
    int bad = 0;
    EW_ROUNDS_U(i0, S, n, kUpdU) {
        if (!have) load(i0, S);
        have = false;
#pragma unroll
        for (int u = 0; u < kUpdU; ++u) {
            const int64_t i = i0 + u * S;
            if (i >= n) continue;
            if (mode != 2) st_hint(x + i, __dadd_rn(xv[u], __dmul_rn(alpha, pv[u])), first);
            if (mode == 1) continue;
            // mode 0: r - alpha q; mode 2: b - Ax (rv holds b)
            const double ri = mode == 0 ? __dsub_rn(rv[u], __dmul_rn(alpha, qv[u])) : __dsub_rn(rv[u], qv[u]);
            st_hint(r + i, ri, last);
            bad |= !isfinite(ri);
            const double zi = jacobi ? __ddiv_rn(ri, dv[u]) : ri;
            v[0] = __dadd_rn(v[0], __dmul_rn(ri, ri));
            v[1] = __dadd_rn(v[1], __dmul_rn(ri, zi));
        }
    }
    pdl_trigger();
    if (mode == 1) return;
    if (bad) atomicOr(&st->flags, 1);
    finish<DIST, 2>(v, partials, st, [&](const double (&t)[2]) {
        decide_update(st, t[0], t[1], tol, divergence, hist);
    });
}

// p = z + beta p (cg.cpp:96-99)
// Walks the vectors from the top down: the update kernel just walked them
// bottom up, so the lines it touched last (r, diag, p of the top indices)
// are the ones still in L2 when this kernel starts.
static __global__ void __launch_bounds__(256) p_kernel(double* __restrict__ p, const double* __restrict__ r,
                                                const double* __restrict__ diag, int64_t n, int jacobi,
                                                const State* st) {
    double rv[kU], dv[kU], pv[kU];
    // the first round's diag and p (neither is written by the update
    // kernel this grid follows) go out before the wait; r after it
    const int64_t S0 = (int64_t)gridDim.x * blockDim.x, t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    bool have = t0 < n;
    if (have) {
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int64_t i = n - 1 - (t0 + u * S0);
            dv[u] = i >= 0 && jacobi ? diag[i] : 1.0;
            pv[u] = i >= 0 ? p[i] : 0.0;
        }
    }
    pdl_wait();
    if (st->done) return;
    const double beta = st->beta;
    EW_ROUNDS(i0, S, n) {
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int64_t i = n - 1 - (i0 + u * S);
            const bool ok = i >= 0;
            rv[u] = ok ? r[i] : 0.0;
            if (!have) {
                dv[u] = ok && jacobi ? diag[i] : 1.0;
                pv[u] = ok ? p[i] : 0.0;
            }
        }
        have = false;
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int64_t i = n - 1 - (i0 + u * S);
            if (i < 0) continue;
            const double zi = jacobi ? __ddiv_rn(rv[u], dv[u]) : rv[u];
            p[i] = __dadd_rn(zi, __dmul_rn(beta, pv[u]));
        }
    }
    pdl_trigger();
}

// Ends the SpMV-fused p.q (ew_spmv.cu k1_dot_kernel writes one partial per
// SpMV CTA and exits without a grid-level handshake): CTA f sums partials
// [256 f, 256 f + 256) (one load per thread, fixed tree), then cg::grid_sum
// over these CTAs in `scratch`; its last CTA decides alpha / breakdown, or
// stores the partition total in loc[slot] for a partitioned solve.
static __global__ void __launch_bounds__(kRedBlock) dot_final_kernel(const double* __restrict__ part, unsigned n,
                                                                     double* scratch, unsigned* tickets, State* st,
                                                                     int dist, int slot) {
    pdl_wait();
    // the update kernel may launch now: it loads its first vectors while
    // this grid sums (it reads alpha only after its own wait)
    pdl_trigger();
    if (st->done) return;  // uniform across the grid
    const unsigned i = blockIdx.x * kRedBlock + threadIdx.x;
    double v[1] = {i < n ? part[i] : 0.0};
    block_sum<1>(v);
    double total;
    if (!grid_sum(v[0], scratch, tickets, &st->ticket, total)) return;
    if (dist) {
        st->loc[slot] = total;
        if (slot == 0) st->loc[1] = 0.0;
    } else {
        decide_pq(st, total);
    }
}

// partials / tickets the fused p.q of a plain SpMV grid of `blocks` CTAs needs
inline size_t dot_final_blocks(int64_t blocks) { return static_cast<size_t>((blocks + kRedBlock - 1) / kRedBlock); }
// (one partial per SpMV warp: 8 per 256-thread CTA)
inline size_t dot_partials(int64_t blocks) {
    return static_cast<size_t>(8 * blocks) + grid_sum_partials(static_cast<int64_t>(dot_final_blocks(8 * blocks)));
}
inline size_t dot_tickets(int64_t blocks) {
    return grid_sum_tickets(static_cast<int64_t>(dot_final_blocks(8 * blocks)));
}

// DIST: sum the all-gathered partition totals in rank order, then decide.
__device__ __forceinline__ void finalize_body(int what, const double* gathered, int nparts, double tol,
                                              double divergence, State* st, double* hist) {
    if (what != kBnorm && what != kStart && st->done) return;
    double t0 = 0.0, t1 = 0.0;
    for (int g = 0; g < nparts; ++g) {
        t0 = __dadd_rn(t0, gathered[2 * g]);
        t1 = __dadd_rn(t1, gathered[2 * g + 1]);
    }
    switch (what) {
        case kBnorm: decide_bnorm(st, t0); break;
        case kStart: decide_start(st, t0, t1, tol, hist); break;
        case kPq: decide_pq(st, __dadd_rn(t0, t1)); break;  // interior + boundary row sets
        default: decide_update(st, t0, t1, tol, divergence, hist); break;
    }
}

static __global__ void finalize_kernel(int what, const double* __restrict__ gathered, int nparts, double tol,
                                       double divergence, State* st, double* hist) {
    finalize_body(what, gathered, nparts, tol, divergence, st, hist);
}

inline unsigned red_grid(int64_t n) {
    int64_t g = (n + kRedBlock - 1) / kRedBlock;
    if (g > kRedGridMax) g = kRedGridMax;
    return static_cast<unsigned>(g < 1 ? 1 : g);
}

// Grid-stride kernels: exactly one wave of resident CTAs (SM count x
// occupancy), so no partial last wave idles half the GPU; capped by the
// partial-sum buffer and by the work.
template <typename Kernel>
unsigned resident_grid(Kernel kernel, int block, int64_t n) {
    static thread_local int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, 0) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    int64_t g = static_cast<int64_t>(sms) * per_sm;
    if (g > kRedGridMax) g = kRedGridMax;
    const int64_t need = (n + block - 1) / block;
    if (g > need) g = need;
    return static_cast<unsigned>(g < 1 ? 1 : g);
}

inline unsigned stream_grid(int64_t n) {
    int64_t g = (n + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    return static_cast<unsigned>(g < 1 ? 1 : g);
}

}  // namespace cg
}  // namespace ew

// ELL-WARP SpMV kernels for sm_100a (paper Listings 1 and 2, PAPER.md:339-362,
// 464-511; reference emulation warp_spmv.cpp:9-126).
//
// HBM-bound by design (0.16 flop/byte): each layout warp streams its own
// contiguous slab of values (8 B) and int32 columns (4 B), column-major so
// the 32 lanes of a step read 256 B + 128 B contiguous. The matrix stream is
// loaded with L1::no_allocate + an L2 evict_first policy so the gathered x
// vector keeps its L2 residency; x is read through the read-only path.
//
// Arithmetic is bit-identical to the reference: each lane sums
// values[s]*x[col[s]] from 0.0 over all maxrows steps of its warp (padding
// included), with the multiply and the add rounded separately (no FMA), and
// K2 combines lane partials with the reference's ascending-stride pairwise
// tree (stride 1, 2, 4, ...), done here with __shfl_down_sync.
#include <cstdlib>
#include <mutex>
#include <string>

#include "ew_cg.cuh"

namespace ew {

namespace {

// CTA-size A/B knob: a multiple of 32 in [32, 256] (the kernels index one
// partial per warp and carry __launch_bounds__(256)); anything else -> dflt.
int cta_size_knob(const char* e, int dflt) {
    if (!e) return dflt;
    const int v = std::atoi(e);
    return (v >= 32 && v <= 256 && v % 32 == 0) ? v : dflt;
}

__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ double ld_stream(const double* p, uint64_t pol) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
                 : "=d"(v)
                 : "l"(p), "l"(pol));
    return v;
}

__device__ __forceinline__ int32_t ld_stream(const int32_t* p, uint64_t pol) {
    int32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;"
                 : "=r"(v)
                 : "l"(p), "l"(pol));
    return v;
}

__device__ __forceinline__ double madd(double acc, double a, double b) {
    return __dadd_rn(acc, __dmul_rn(a, b));  // two roundings, as the reference
}

struct K1Args {
    const double* values;
    const int32_t* cols;
    const int64_t* woff;
    const int32_t* maxrows;
    const int32_t* slen;  // !SORTED only
    const int32_t* fwd;   // SCATTER only
    const double* x;
    double* y;
    const int* done;
    int64_t nrows, n_active;
    int32_t ws, ws_log2;
    const double* xg;  // SPLIT_X: columns >= nown read xg[c - nown] (a ghost tail)
    int32_t nown;
    const uint16_t* cols16;   // COMPACT: 16-bit column offsets (LayoutData::cols16)
    const int32_t* col_base;  // COMPACT: per-warp smallest column
    const int32_t* widx;      // INDIRECT: the layout warps to run, thread i -> warp widx[i / ws]
    int64_t nidx;             // INDIRECT: entries of widx
    // GROUPED (LayoutData::grouped): shared column lists
    const uint8_t* lane_grp;
    const uint8_t* ngrp;
    const int64_t* goff;
    const int32_t* gcols;
    const uint16_t* gcols16;
    int64_t row_lo;  // k1_kernel (!INDIRECT): thread i runs sorted row row_lo + i (the tail of a head split)
    const int64_t* col_shift;  // shrunk compact layouts: wide warp w's int32 columns at cols + col_shift[w]
};

// The int32 columns of (wide) layout warp w, indexed by slot.
__device__ __forceinline__ const int32_t* wide_cols(const K1Args& a, int64_t w) {
    return a.col_shift ? a.cols + a.col_shift[w] : a.cols;
}

__device__ __forceinline__ uint16_t ld_stream(const uint16_t* p, uint64_t pol) {
    uint16_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u16 %0, [%1], %2;"
                 : "=h"(v)
                 : "l"(p), "l"(pol));
    return v;
}

// Column sources of a lane sum: the int32 slab, or the compact one (16-bit
// offsets from the warp's smallest column, 0xFFFF = padding = column 0).
__device__ __forceinline__ auto cols32(const int32_t* __restrict__ cols) {
    return [cols](int64_t i, uint64_t pol) { return ld_stream(cols + i, pol); };
}
__device__ __forceinline__ auto cols16(const uint16_t* __restrict__ c16, int32_t base) {
    return [c16, base](int64_t i, uint64_t pol) {
        const uint16_t d = ld_stream(c16 + i, pol);
        return d == 0xFFFFu ? 0 : base + static_cast<int32_t>(d);
    };
}

// Serial lane sum over j in [0, mx) at stride `step` from slot s, unrolled by
// 8 so eight value/column loads and then eight x gathers are in flight per
// thread before the (order-preserving) accumulation chain consumes them; the
// last mx % 4 steps go in one predicated block (two round trips, not two per
// step).
template <typename ColLoad, typename XLoad>
__device__ __forceinline__ double lane_sum_x(const double* __restrict__ vals, ColLoad ld_c, XLoad ld_x, int64_t s,
                                             int64_t step, int32_t mx, uint64_t pol) {
    double sum = 0.0;
    int32_t j = 0;
    for (; j + 8 <= mx; j += 8) {
        int32_t c[8];
        double v[8], xv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) c[u] = ld_c(s + u * step, pol);
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = ld_stream(vals + s + u * step, pol);
#pragma unroll
        for (int u = 0; u < 8; ++u) xv[u] = ld_x(c[u]);
#pragma unroll
        for (int u = 0; u < 8; ++u) sum = madd(sum, v[u], xv[u]);
        s += 8 * step;
    }
    if (j + 4 <= mx) {
        int32_t c[4];
        double v[4], xv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) c[u] = ld_c(s + u * step, pol);
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = ld_stream(vals + s + u * step, pol);
#pragma unroll
        for (int u = 0; u < 4; ++u) xv[u] = ld_x(c[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u) sum = madd(sum, v[u], xv[u]);
        s += 4 * step;
        j += 4;
    }
    // last 0..3 steps predicated, so their loads are in flight together too
    const int32_t rem = mx - j;
    if (rem > 0) {
        int32_t c[3];
        double v[3], xv[3];
#pragma unroll
        for (int u = 0; u < 3; ++u)
            if (u < rem) c[u] = ld_c(s + u * step, pol);
#pragma unroll
        for (int u = 0; u < 3; ++u)
            if (u < rem) v[u] = ld_stream(vals + s + u * step, pol);
#pragma unroll
        for (int u = 0; u < 3; ++u)
            if (u < rem) xv[u] = ld_x(c[u]);
#pragma unroll
        for (int u = 0; u < 3; ++u)
            if (u < rem) sum = madd(sum, v[u], xv[u]);
    }
    return sum;
}

__device__ __forceinline__ double lane_sum(const double* __restrict__ vals, const int32_t* __restrict__ cols,
                                           const double* __restrict__ x, int64_t s, int64_t step, int32_t mx,
                                           uint64_t pol) {
    // x gathers: read-only path with an L2 evict_last hint, so the vector
    // outlives the evict_first matrix stream in L2 (gather-bound layouts:
    // config 4's SpMV 155.2 -> 153.7 us; the stream form below keeps __ldg,
    // where the hint cost 0.5% on config 2)
    uint64_t keep;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
    return lane_sum_x(vals, cols32(cols), [x, keep](int32_t c) {
        double v;
        asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(x + c), "l"(keep));
        return v;
    }, s, step, mx, pol);
}

__device__ __forceinline__ double lane_sum_ldg(const double* __restrict__ vals, const int32_t* __restrict__ cols,
                                               const double* __restrict__ x, int64_t s, int64_t step, int32_t mx,
                                               uint64_t pol) {
    return lane_sum_x(vals, cols32(cols), [x](int32_t c) { return __ldg(x + c); }, s, step, mx, pol);
}

// x split in two arrays: owned columns [0, nown) in x, the ghost tail in xg
// (a partition's local columns; the caller's x needs no copy).
__device__ __forceinline__ double lane_sum_split(const double* __restrict__ vals, const int32_t* __restrict__ cols,
                                                 const double* __restrict__ x, const double* __restrict__ xg,
                                                 int32_t nown, int64_t s, int64_t step, int32_t mx, uint64_t pol) {
    return lane_sum_x(vals, cols32(cols), [x, xg, nown](int32_t c) { return c < nown ? __ldg(x + c) : __ldg(xg + (c - nown)); },
                      s, step, mx, pol);
}

// lane_sum_x with the columns read from a grouped list: step j's column at
// gc(g + j * ng) (the values still at s + j * step). Same loads in flight,
// same order of the adds.
template <typename ColLoad, typename XLoad>
__device__ __forceinline__ double lane_sum_gx(const double* __restrict__ vals, ColLoad gc, XLoad ld_x, int64_t s,
                                              int64_t step, int64_t g, int32_t ng, int32_t mx, uint64_t pol) {
    double sum = 0.0;
    int32_t j = 0;
    for (; j + 8 <= mx; j += 8) {
        int32_t c[8];
        double v[8], xv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) c[u] = gc(g + u * ng, pol);
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = ld_stream(vals + s + u * step, pol);
#pragma unroll
        for (int u = 0; u < 8; ++u) xv[u] = ld_x(c[u]);
#pragma unroll
        for (int u = 0; u < 8; ++u) sum = madd(sum, v[u], xv[u]);
        s += 8 * step;
        g += 8 * ng;
    }
    if (j + 4 <= mx) {
        int32_t c[4];
        double v[4], xv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) c[u] = gc(g + u * ng, pol);
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = ld_stream(vals + s + u * step, pol);
#pragma unroll
        for (int u = 0; u < 4; ++u) xv[u] = ld_x(c[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u) sum = madd(sum, v[u], xv[u]);
        s += 4 * step;
        g += 4 * ng;
        j += 4;
    }
    const int32_t rem = mx - j;
    if (rem > 0) {
        int32_t c[3];
        double v[3], xv[3];
#pragma unroll
        for (int u = 0; u < 3; ++u)
            if (u < rem) c[u] = gc(g + u * ng, pol);
#pragma unroll
        for (int u = 0; u < 3; ++u)
            if (u < rem) v[u] = ld_stream(vals + s + u * step, pol);
#pragma unroll
        for (int u = 0; u < 3; ++u)
            if (u < rem) xv[u] = ld_x(c[u]);
#pragma unroll
        for (int u = 0; u < 3; ++u)
            if (u < rem) sum = madd(sum, v[u], xv[u]);
    }
    return sum;
}

// One K1 lane sum of sorted row p (layout warp w) from the grouped column
// lists: 16-bit offsets when the layout is compact (its wide warps read their
// own int32 columns), else int32. x gathers with the evict_last hint.
template <bool COMPACT>
__device__ __forceinline__ double k1_row_grouped(const K1Args& a, int64_t w, int64_t p, int64_t s, int32_t mx,
                                                 uint64_t pol) {
    const int64_t g = a.goff[w] + a.lane_grp[p];
    const int32_t ng = a.ngrp[w];
    const double* x = a.x;
    uint64_t keep;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
    auto ldx = [x, keep](int32_t c) {
        double v;
        asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(x + c), "l"(keep));
        return v;
    };
    if (COMPACT) {
        const int32_t base = a.col_base[w];
        if (base < 0) return lane_sum(a.values, wide_cols(a, w), a.x, s, a.ws, mx, pol);  // a wide warp: own int32 columns
        const uint16_t* g16 = a.gcols16;
        return lane_sum_gx(a.values, [g16, base](int64_t i, uint64_t pl) {
            const uint16_t d = ld_stream(g16 + i, pl);
            return d == 0xFFFFu ? 0 : base + static_cast<int32_t>(d);
        }, ldx, s, a.ws, g, ng, mx, pol);
    }
    const int32_t* g32 = a.gcols;
    return lane_sum_gx(a.values, [g32](int64_t i, uint64_t pl) { return ld_stream(g32 + i, pl); }, ldx, s, a.ws, g,
                       ng, mx, pol);
}

// One K1 lane sum of layout warp w. COMPACT: 16-bit columns (LayoutData::
// cols16: 10 instead of 12 bytes per slot streamed) for the warps that have
// them; x gathers with the evict_last hint either way.
template <bool COMPACT>
__device__ __forceinline__ double k1_row(const K1Args& a, int64_t w, int64_t s, int64_t step, int32_t mx,
                                         uint64_t pol) {
    if (COMPACT) {
        const int32_t base = a.col_base[w];  // < 0: this warp's columns span too far, int32 slab
        if (base >= 0) {
            const double* x = a.x;
            uint64_t keep;
            asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
            return lane_sum_x(a.values, cols16(a.cols16, base), [x, keep](int32_t c) {
                double v;
                asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(x + c), "l"(keep));
                return v;
            }, s, step, mx, pol);
        }
        return lane_sum(a.values, wide_cols(a, w), a.x, s, step, mx, pol);
    }
    return lane_sum(a.values, a.cols, a.x, s, step, mx, pol);
}

// K1 / K1r / K1rs (warp_spmv.cpp:9-60): one thread per sorted row position.
// SCATTER stores y[Pinv[p]] (K1); otherwise y[p] in sorted numbering.
#ifndef EW_K1C_MINB
#define EW_K1C_MINB 5
#endif
// grouped int32 layouts (config 5): plain and grid-stride forms
#ifndef EW_K1G_STREAM_MINB
#define EW_K1G_STREAM_MINB 8
#endif
#ifndef EW_K1G_MINB
#define EW_K1G_MINB 8
#endif
#ifndef EW_K1P_MINB
#define EW_K1P_MINB 8
#endif
// INDIRECT runs only the layout warps listed in widx (the host-buffer
// pipeline's stages, ew_kernel.cu): the same warps, lanes and padding as the
// whole-layout launch, so the same row sums.
template <bool SORTED, bool SCATTER, bool ROW_MAJOR, bool SPLIT_X = false, bool COMPACT = false,
          bool INDIRECT = false, bool GROUPED = false>
__global__ void __launch_bounds__(256, COMPACT ? EW_K1C_MINB : (GROUPED ? EW_K1G_MINB : EW_K1P_MINB))
    k1_kernel(K1Args a) {
    pdl_wait();
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (!INDIRECT) p += a.row_lo;
    if (INDIRECT) {
        const int64_t i = p >> a.ws_log2;
        if (i >= a.nidx) return;
        p = (int64_t(a.widx[i]) << a.ws_log2) | (p & (a.ws - 1));
    }
    if (p >= a.nrows || (a.done && *a.done)) return;
    const uint64_t pol = evict_first_policy();
    // the scatter target is loaded with the metadata, not after the row sum
    const int64_t target = SCATTER ? a.fwd[p] : p;
    double sum = 0.0;
    const bool active = SORTED ? p < a.n_active : a.slen[p] > 0;
    if (active) {
        const int64_t w = p >> a.ws_log2;
        const int32_t lane = static_cast<int32_t>(p & (a.ws - 1));
        const int32_t mx = a.maxrows[w];
        const int64_t s = a.woff[w] + (ROW_MAJOR ? int64_t(lane) * mx : lane);
        if (GROUPED)
            sum = k1_row_grouped<COMPACT>(a, w, p, s, mx, pol);
        else
            sum = SPLIT_X ? lane_sum_split(a.values, a.cols, a.x, a.xg, a.nown, s, ROW_MAJOR ? 1 : a.ws, mx, pol)
                          : k1_row<COMPACT>(a, w, s, ROW_MAJOR ? 1 : a.ws, mx, pol);
    }
    a.y[target] = sum;
    pdl_trigger();
}

// The same K1 in grid-stride form, for layouts well beyond L2 (the launch
// grid is still one CTA per 256 rows, so the body runs once per thread).
// ptxas schedules this form differently under the 32-register cap: it keeps
// the row index and store address out of registers across the lane loop
// (spilled to L1) and issues all eight column loads of a block before the
// first x gather. On HBM-bound matrices with long rows that is +4.5%
// (config 2, 44 slots per row: 170.5 -> 163 us, 0.95 -> 0.995 of HBM); on
// L2-resident ones the spill traffic costs more than it gains (config 1:
// 7.6 -> 9.1 us), and short-row gather-bound ones (config 4, 15 per row)
// lose 1-5%, so layout_spmv picks by size and row length (the CG's fused
// p.q kernel likewise: config-2-sized slab CG +4.8%). Same arithmetic,
// bit-identical results. Layouts with 16-bit columns (compact_layout) run the
// plain form instead: with the narrower column loads the stream form spills
// more (221 us cold on config 2) and the plain one wins (158.0 us vs 163.6).
template <bool SORTED, bool SCATTER, bool SPLIT_X = false, bool GROUPED = false>
__global__ void __launch_bounds__(256, GROUPED ? EW_K1G_STREAM_MINB : 8) k1_stream_kernel(K1Args a) {
    pdl_wait();
    if (a.done && *a.done) return;
    const uint64_t pol = evict_first_policy();
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < a.nrows;
         p += (int64_t)gridDim.x * blockDim.x) {
        double sum = 0.0;
        const bool active = SORTED ? p < a.n_active : a.slen[p] > 0;
        if (active) {
            const int64_t w = p >> a.ws_log2;
            const int32_t lane = static_cast<int32_t>(p & (a.ws - 1));
            const int32_t mx = a.maxrows[w];
            const int64_t s = a.woff[w] + lane;
            if (GROUPED)
                sum = k1_row_grouped<false>(a, w, p, s, mx, pol);
            else
                sum = SPLIT_X ? lane_sum_split(a.values, a.cols, a.x, a.xg, a.nown, s, a.ws, mx, pol)
                              : lane_sum_ldg(a.values, a.cols, a.x, s, a.ws, mx, pol);
        }
        a.y[SCATTER ? a.fwd[p] : p] = sum;
    }
    pdl_trigger();
}

// K1 for layouts with few, long rows (the FEM matrices of the paper's suite
// at Table 2 sizes: 36k-220k rows of 20-120 entries, i.e. under one wave of
// one-thread-per-row CTAs, each thread walking its row 8 slots per round
// trip). One CTA of H warps per layout warp (ws = 32): every warp loads and
// multiplies its share of each chunk of 8H steps (H times the loads in
// flight), the products go to shared memory, and warp 0 adds them in step
// order. Same products (v * x[c], padding included), same sequential sum per
// row as k1_kernel: bit-identical y.
#ifndef EW_COOP8_MINB
#define EW_COOP8_MINB 4
#endif
#ifndef EW_COOP4_MINB
#define EW_COOP4_MINB 8
#endif
#ifndef EW_COOP2_MINB
#define EW_COOP2_MINB 16
#endif
template <bool SCATTER, bool COMPACT, int H>
__global__ void __launch_bounds__(32 * H, H == 8 ? EW_COOP8_MINB : (H == 4 ? EW_COOP4_MINB : EW_COOP2_MINB))
    k1_coop_kernel(K1Args a) {
    constexpr int C = 8 * H;
    __shared__ double prod[2][C][32];
    pdl_wait();
    if (a.done && *a.done) return;  // uniform across the grid
    const int64_t w = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t p = (w << 5) + lane;
    const int32_t mx = __ldg(a.maxrows + w);
    const int64_t wo = __ldg(a.woff + w);
    const int32_t base = COMPACT ? __ldg(a.col_base + w) : -1;
    int64_t target = p;
    if (SCATTER && warp == 0 && p < a.nrows) target = a.fwd[p];
    const uint64_t pol = evict_first_policy();
    uint64_t keep;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
    double acc = 0.0;
    const int nchunks = (mx + C - 1) / C;
    for (int c = 0; c < nchunks; ++c) {
        const int j0 = c * C + warp * 8;
        const int cnt = min(8, mx - j0);
        if (cnt > 0) {
            const int64_t s0 = wo + int64_t(j0) * 32 + lane;
            int32_t col[8];
            double v[8], xv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if (u < cnt) {
                    if (COMPACT && base >= 0) {
                        const uint16_t d = ld_stream(a.cols16 + s0 + u * 32, pol);
                        col[u] = d == 0xFFFFu ? 0 : base + static_cast<int32_t>(d);
                    } else {
                        col[u] = ld_stream((COMPACT ? wide_cols(a, w) : a.cols) + s0 + u * 32, pol);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (u < cnt) v[u] = ld_stream(a.values + s0 + u * 32, pol);
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (u < cnt)
                    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;"
                                 : "=d"(xv[u])
                                 : "l"(a.x + col[u]), "l"(keep));
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (u < cnt) prod[c & 1][warp * 8 + u][lane] = __dmul_rn(v[u], xv[u]);
        }
        __syncthreads();
        if (warp == 0) {
            const int n = min(C, mx - c * C);
#pragma unroll 8
            for (int j = 0; j < n; ++j) acc = __dadd_rn(acc, prod[c & 1][j][lane]);
        }
    }
    if (warp == 0 && p < a.nrows) a.y[target] = p < a.n_active ? acc : 0.0;
    pdl_trigger();
}

// K1 for the very long rows at the head of a power-law layout (the head of a
// head split, layout_spmv): one 1024-thread CTA per layout warp. Warps 1-31
// load and multiply 8 steps each of every chunk of 248 steps, warp 0 adds
// the products in step order; two chunk buffers in shared memory change
// hands through named barriers (FULL b: the producers arrive, the adder
// waits; EMPTY b: the adder arrives, the producers wait before reusing b),
// so the adds of chunk c overlap the loads of chunk c + 1. Same products,
// same sequential sum per row as k1_kernel: bit-identical y.
constexpr int kLongProducers = 31;
constexpr int kLongChunk = 8 * kLongProducers;
constexpr size_t kLongSmem = 2 * kLongChunk * 32 * sizeof(double);

__device__ __forceinline__ void named_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int count) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// FORM: the column form the layout keeps -- 0 int32, 1 16-bit offsets (wide
// warps: their int32 columns), 2 grouped int32 lists, 3 grouped 16-bit.
template <bool SCATTER, int FORM>
__global__ void __launch_bounds__(1024, 1) k1_long_kernel(K1Args a) {
    extern __shared__ double prod[];  // [2][kLongChunk][32]
    if (a.done && *a.done) return;    // uniform across the grid
    const int64_t w = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t p = (w << 5) + lane;
    const int32_t mx = __ldg(a.maxrows + w);
    const int64_t wo = __ldg(a.woff + w);
    constexpr bool kCompact = FORM == 1 || FORM == 3, kGrouped = FORM >= 2;
    const int32_t base = kCompact ? __ldg(a.col_base + w) : 0;
    const int32_t* wc = kCompact ? wide_cols(a, w) : a.cols;
    const int64_t g0 = kGrouped && p < a.nrows ? a.goff[w] + a.lane_grp[p] : 0;
    const int32_t ng = kGrouped ? a.ngrp[w] : 0;
    const int nchunks = (mx + kLongChunk - 1) / kLongChunk;
    if (warp == 0) {
        const int64_t target = SCATTER && p < a.nrows ? a.fwd[p] : p;
        double acc = 0.0;
        for (int c = 0; c < nchunks; ++c) {
            const int b = c & 1;
            named_sync(1 + b, 1024);  // chunk c is in buffer b
            const double* buf = prod + b * (kLongChunk * 32);
            const int n = min(kLongChunk, mx - c * kLongChunk);
#pragma unroll 8
            for (int j = 0; j < n; ++j) acc = __dadd_rn(acc, buf[j * 32 + lane]);
            if (c + 2 < nchunks) named_arrive(3 + b, 1024);  // buffer b free for chunk c + 2
        }
        if (p < a.nrows) a.y[target] = p < a.n_active ? acc : 0.0;
    } else {
        const uint64_t pol = evict_first_policy();
        uint64_t keep;
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
        const int q = warp - 1;
        for (int c = 0; c < nchunks; ++c) {
            const int b = c & 1;
            if (c >= 2) named_sync(3 + b, 1024);  // the adder is done with chunk c - 2
            const int j0 = c * kLongChunk + q * 8;
            const int cnt = min(8, mx - j0);
            if (cnt > 0) {
                const int64_t s0 = wo + int64_t(j0) * 32 + lane;
                int32_t col[8];
                double v[8], xv[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    if (u >= cnt) continue;
                    const int64_t sl = s0 + u * 32;
                    if (FORM == 0 || (kCompact && base < 0)) {
                        col[u] = ld_stream(wc + sl, pol);
                    } else if (FORM == 2) {
                        col[u] = p < a.nrows ? ld_stream(a.gcols + g0 + int64_t(j0 + u) * ng, pol) : 0;
                    } else {
                        const uint16_t d = FORM == 1 ? ld_stream(a.cols16 + sl, pol)
                                           : p < a.nrows ? ld_stream(a.gcols16 + g0 + int64_t(j0 + u) * ng, pol)
                                                         : uint16_t(0xFFFF);
                        col[u] = d == 0xFFFFu ? 0 : base + static_cast<int32_t>(d);
                    }
                }
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (u < cnt) v[u] = ld_stream(a.values + s0 + u * 32, pol);
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (u < cnt)
                        asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;"
                                     : "=d"(xv[u])
                                     : "l"(a.x + col[u]), "l"(keep));
                double* buf = prod + b * (kLongChunk * 32);
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (u < cnt) buf[(q * 8 + u) * 32 + lane] = __dmul_rn(v[u], xv[u]);
            }
            named_arrive(1 + b, 1024);
        }
    }
}

template <bool SCATTER>
void launch_k1_long(const K1Args& a, int64_t nwarps, int form, cudaStream_t s) {
    const unsigned g = static_cast<unsigned>(nwarps);
    if (form == 0) k1_long_kernel<SCATTER, 0><<<g, 1024, kLongSmem, s>>>(a);
    else if (form == 1) k1_long_kernel<SCATTER, 1><<<g, 1024, kLongSmem, s>>>(a);
    else if (form == 2) k1_long_kernel<SCATTER, 2><<<g, 1024, kLongSmem, s>>>(a);
    else k1_long_kernel<SCATTER, 3><<<g, 1024, kLongSmem, s>>>(a);
    EW_CUDA_CHECK(cudaGetLastError());
    launched("k1_long_kernel");
}

// ---- the same K1 with the warp's slab staged by the bulk-copy engine -------
// k1_coop_kernel's loads (8 column + 8 value loads per lane and warp per
// chunk, then the gathers) replaced by cp.async.bulk copies of whole chunks
// of the layout warp's slab into shared memory (the slab is contiguous and
// 256 / 128-byte aligned per warp, warp_layout.cpp:12-16), two chunks in
// flight ahead of the one being multiplied, completion on an mbarrier: the
// threads only gather x and multiply. Same products, same order: identical y.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

template <bool SCATTER, int H>
__global__ void __launch_bounds__(32 * H) k1_bulk_kernel(K1Args a) {
    constexpr int C = 8 * H;  // steps per chunk
    extern __shared__ __align__(128) unsigned char k1b_smem[];
    double* vals = reinterpret_cast<double*>(k1b_smem);                      // [2][C][32]
    int32_t* cols = reinterpret_cast<int32_t*>(k1b_smem + 2 * C * 32 * 8);  // [2][C][32]
    __shared__ __align__(8) uint64_t bar[2];
    pdl_wait();
    if (a.done && *a.done) return;  // uniform across the grid
    const int64_t w = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t p = (w << 5) + lane;
    const int32_t mx = __ldg(a.maxrows + w);
    const int64_t wo = __ldg(a.woff + w);
    const int nchunks = (mx + C - 1) / C;
    const uint64_t pol = evict_first_policy();
    auto issue = [&](int c) {  // one thread: chunk c into stage c & 1
        const int st = c & 1;
        const int cnt = min(C, mx - c * C);
        const uint32_t vb = static_cast<uint32_t>(cnt) * 256u, cb = static_cast<uint32_t>(cnt) * 128u;
        mbar_expect_tx(&bar[st], vb + cb);
        const int64_t s0 = wo + int64_t(c) * C * 32;
        bulk_g2s(vals + st * C * 32, a.values + s0, vb, &bar[st], pol);
        bulk_g2s(cols + st * C * 32, a.cols + s0, cb, &bar[st], pol);
    };
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int c = 0; c < min(2, nchunks); ++c) issue(c);
    }
    int64_t target = p;
    if (SCATTER && warp == 0 && p < a.nrows) target = a.fwd[p];
    __syncthreads();
    uint64_t keep;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
    double acc = 0.0;
    for (int c = 0; c < nchunks; ++c) {
        const int st = c & 1;
        mbar_wait(&bar[st], (c >> 1) & 1);
        const int j0 = warp * 8, cnt = min(8, mx - c * C - j0);
        double* v = vals + st * C * 32;
        const int32_t* cl = cols + st * C * 32;
        if (cnt > 0) {
            double xv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (u < cnt)
                    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;"
                                 : "=d"(xv[u])
                                 : "l"(a.x + cl[(j0 + u) * 32 + lane]), "l"(keep));
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (u < cnt) v[(j0 + u) * 32 + lane] = __dmul_rn(v[(j0 + u) * 32 + lane], xv[u]);
        }
        __syncthreads();
        if (warp == 0) {
            const int n = min(C, mx - c * C);
#pragma unroll 8
            for (int j = 0; j < n; ++j) acc = __dadd_rn(acc, v[j * 32 + lane]);
            __syncwarp();
            if (lane == 0 && c + 2 < nchunks) {
                // the generic-proxy reads / writes of this stage come before
                // the bulk copy's writes into it
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue(c + 2);
            }
        }
    }
    if (warp == 0 && p < a.nrows) a.y[target] = p < a.n_active ? acc : 0.0;
    pdl_trigger();
}

template <bool SCATTER>
void launch_k1_bulk(const K1Args& a, int64_t nwarps, int h, cudaStream_t s) {
    const unsigned g = static_cast<unsigned>(nwarps);
    auto go = [&](auto kernel, int hh) {
        const int smem = 2 * 8 * hh * 32 * 12;
        static std::once_flag once[3];
        std::call_once(once[hh == 2 ? 0 : (hh == 4 ? 1 : 2)],
                       [&] { cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); });
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(g);
        cfg.blockDim = dim3(32 * hh);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = pdl_enabled() ? 1 : 0;
        cuda_check(cudaLaunchKernelEx(&cfg, kernel, a), "cudaLaunchKernelEx(k1_bulk_kernel)");
    };
    if (h == 2) go(k1_bulk_kernel<SCATTER, 2>, 2);
    else if (h == 4) go(k1_bulk_kernel<SCATTER, 4>, 4);
    else go(k1_bulk_kernel<SCATTER, 8>, 8);
    launched("k1_bulk_kernel");
}

// Warps per CTA of k1_coop_kernel for a layout, 0: the plain kernel. Sorted,
// column-major ws = 32 int32-column layouts with under one wave of
// one-thread-per-row CTAs (148 SMs x 2048 threads), unless they are over
// half a wave of rows of at most 32 entries. H trades the chunks the
// longest warp walks in sequence (ceil(max_mx / 8H)) against resident CTAs
// (~32 / H per SM): layouts with a row over 96 entries take 8, small ones
// (<= 8 CTAs per SM at H = 4) 4, the rest 2 -- the best or within 5% of the
// best H on every config-3 matrix (H = 2 / 4 / 8 sweep on B200). 16-bit-column
// layouts (over 64 MB) keep their 64-thread-CTA form, which wins there (ship,
// spheres, windtunnel). EW_K1_COOP=0 turns it off, =2/4/8 fixes H (A/B runs).
int coop_warps(const LayoutData& l) {
    static const int mode = [] {
        const char* e = std::getenv("EW_K1_COOP");
        return e ? std::atoi(e) : 1;
    }();
    if (!mode || l.kind != EW_LAYOUT_K1 || l.row_major || !l.sorted || l.imported || l.ws != 32 || l.nwarps == 0)
        return 0;
    if (mode == 2 || mode == 4 || mode == 8) return mode;  // A/B: a fixed H
    if (l.nrows > int64_t{148} * 2048 || l.compact) return 0;
    // over half a wave of short rows only (config 1: 262k rows of 5-15):
    // the plain kernel's chains are short and its grid fills the GPU
    // (5.8 us vs 10.7 us for H = 2)
    if (l.nrows > int64_t{148} * 1024 && l.max_mx > 0 && l.max_mx <= 32) return 0;
    if (l.max_mx > 96) return 8;
    if (l.nwarps <= 148 * 8) return 4;
    return 2;
}

template <bool SCATTER>
void launch_k1_coop(const K1Args& a, int64_t nwarps, int h, bool compact, cudaStream_t s) {
    const unsigned g = static_cast<unsigned>(nwarps);
    // (the default shared-memory carveout: a larger one shrinks L1, where
    // half the x gathers hit -- protein 4,973 -> 1,600 GB/s effective)
    auto go = [&](auto kernel, int hh) { launch_pdl(kernel, g, 32 * hh, s, a); };
    if (compact) {
        if (h == 2) go(k1_coop_kernel<SCATTER, true, 2>, 2);
        else if (h == 4) go(k1_coop_kernel<SCATTER, true, 4>, 4);
        else go(k1_coop_kernel<SCATTER, true, 8>, 8);
    } else {
        if (h == 2) go(k1_coop_kernel<SCATTER, false, 2>, 2);
        else if (h == 4) go(k1_coop_kernel<SCATTER, false, 4>, 4);
        else go(k1_coop_kernel<SCATTER, false, 8>, 8);
    }
    launched("k1_coop_kernel");
}

// Layouts whose slabs exceed this stream from HBM, with at least this many
// slots per row: k1_stream_kernel.
constexpr int64_t kStreamSlotBytes = 64ll << 20;
constexpr int64_t kStreamSlotsPerRow = 24;

inline bool streams(const LayoutData& l) {
    static const int force = [] {
        const char* e = std::getenv("EW_K1_FORM");  // A/B runs: "stream" / "plain"
        return e ? (std::string(e) == "stream" ? 1 : 0) : -1;
    }();
    if (force >= 0) return force == 1;
    return l.nslots * 12 > kStreamSlotBytes && l.nslots >= kStreamSlotsPerRow * l.nrows;
}

// K1 with the CG's p.q fused in (cg.cpp:72): the operator input x is p, so
// each row adds x[target] * y[target] to its CTA's fixed-order partial;
// cg::dot_final_kernel sums the partials and decides. The CTA only stores
// its partial: no fence or atomic holds it past its last row.
template <bool SORTED, bool SCATTER, bool COMPACT = false, bool GROUPED = false>
__global__ void __launch_bounds__(256, COMPACT ? EW_K1C_MINB : (GROUPED ? EW_K1G_MINB : EW_K1P_MINB))
    k1_dot_kernel(K1Args a, double* __restrict__ partials) {
    pdl_wait();
    if (a.done && *a.done) return;  // uniform across the grid
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    double v[1] = {0.0};
    if (p < a.nrows) {
        const uint64_t pol = evict_first_policy();
        double sum = 0.0;
        // target and p[target] loaded with the metadata, not after the row sum
        const int64_t t = SCATTER ? a.fwd[p] : p;
        const double xt = a.x[t];
        const bool active = SORTED ? p < a.n_active : a.slen[p] > 0;
        if (active) {
            const int64_t w = p >> a.ws_log2;
            const int32_t lane = static_cast<int32_t>(p & (a.ws - 1));
            sum = GROUPED ? k1_row_grouped<COMPACT>(a, w, p, a.woff[w] + lane, a.maxrows[w], pol)
                          : k1_row<COMPACT>(a, w, a.woff[w] + lane, a.ws, a.maxrows[w], pol);
        }
        a.y[t] = sum;
        v[0] = __dmul_rn(xt, sum);
    }
    pdl_trigger();
    // one partial per warp (fixed shuffle tree): no CTA-wide barrier holds
    // the CTA past its slowest warp
    const double wsum = cg::warp_sum(v[0]);
    if ((threadIdx.x & 31) == 0) partials[blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)] = wsum;
}

// k1_dot_kernel in the grid-stride form of k1_stream_kernel (large long-row layouts).
template <bool SORTED, bool SCATTER, bool GROUPED = false>
__global__ void __launch_bounds__(256, GROUPED ? EW_K1G_STREAM_MINB : 8)
    k1_dot_stream_kernel(K1Args a, double* __restrict__ partials) {
    pdl_wait();
    if (a.done && *a.done) return;  // uniform across the grid
    const uint64_t pol = evict_first_policy();
    double v[1] = {0.0};
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < a.nrows;
         p += (int64_t)gridDim.x * blockDim.x) {
        double sum = 0.0;
        const bool active = SORTED ? p < a.n_active : a.slen[p] > 0;
        if (active) {
            const int64_t w = p >> a.ws_log2;
            const int32_t lane = static_cast<int32_t>(p & (a.ws - 1));
            sum = GROUPED ? k1_row_grouped<false>(a, w, p, a.woff[w] + lane, a.maxrows[w], pol)
                          : lane_sum_ldg(a.values, a.cols, a.x, a.woff[w] + lane, a.ws, a.maxrows[w], pol);
        }
        const int64_t t = SCATTER ? a.fwd[p] : p;
        a.y[t] = sum;
        v[0] = __dadd_rn(v[0], __dmul_rn(a.x[t], sum));
    }
    pdl_trigger();
    const double wsum = cg::warp_sum(v[0]);  // one partial per warp
    if ((threadIdx.x & 31) == 0) partials[blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)] = wsum;
}

struct K2Args {
    const double* values;
    const int32_t* cols;
    const int64_t* woff;
    const int32_t* maxrows;
    const int32_t* reduction;
    const int32_t* rows_offset_warp;
    const int32_t* rows_in_warp;
    const int32_t* slen;
    const int32_t* fwd;
    const double* x;
    double* y;
    const int* done;
    int64_t nwarps, n_active;
    int32_t ws, ws_log2;
};

// K2 / K2r / K2rs (warp_spmv.cpp:62-126) for warp_size <= 32: thread t is lane
// t % ws of layout warp t / ws; `reduction` lanes share a row, each summing a
// contiguous chunk of maxrows slots, then the ascending-stride tree.
// DOT (the CG's fused p.q): each row's leader adds x[target] * y[target];
// one partial per hardware warp, summed by cg::dot_final_kernel.
// 40 registers (6 CTAs of 256 per SM; 48 unbounded, 5 CTAs): the lanes'
// short chains are latency bound, so resident warps pay -- suite, same box:
// harbor 2,948 -> 4,473, protein 3,851 -> 5,297, webbase 1,069 -> 1,303 GB/s
// effective (32 registers / 8 CTAs: 3,647, 4,200, 807).
template <bool SORTED, bool SCATTER, bool DOT = false>
__global__ void __launch_bounds__(256, 6) k2_kernel(K2Args a, double* __restrict__ partials) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t w = t >> a.ws_log2;
    const int32_t lane = static_cast<int32_t>(t & (a.ws - 1));
    pdl_wait();
    if (a.done && *a.done) return;  // uniform across the grid
    const uint64_t pol = evict_first_policy();
    double sum = 0.0;
    int32_t red = 1, tl = 0;
    bool leader = false;
    int64_t pos = 0, target = 0;
    if (w < a.nwarps) {
        // every per-warp field in one round trip (independent loads issued
        // together; ncu: the former chain reduction -> rows_in_warp ->
        // rows_offset_warp -> maxrows held ~30% of a cold launch)
        red = __ldg(a.reduction + w);
        const int32_t riw = __ldg(a.rows_in_warp + w), row0 = __ldg(a.rows_offset_warp + w);
        const int32_t mx = __ldg(a.maxrows + w);
        const int64_t wo = __ldg(a.woff + w);
        const int32_t rl = __ffs(red) - 1;
        const int32_t r = lane >> rl;
        tl = lane & (red - 1);
        if (r < riw) {
            pos = int64_t(row0) + r;
            leader = tl == 0;
            if (SCATTER && leader) target = a.fwd[pos];  // with the metadata, not after the sum
            const bool active = SORTED ? pos < a.n_active : a.slen[pos] > 0;
            if (active) sum = lane_sum(a.values, a.cols, a.x, wo + lane, a.ws, mx, pol);
        }
    }
    const int32_t hw_red = static_cast<int32_t>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(red)));
    for (int32_t st = 1; st < hw_red; st <<= 1) {
        const double o = __shfl_down_sync(0xffffffffu, sum, st);
        if (st < red && (tl & (2 * st - 1)) == 0) sum = __dadd_rn(sum, o);
    }
    if (!SCATTER) target = pos;
    if (leader) a.y[target] = sum;
    pdl_trigger();
    if (DOT) {
        const double part = cg::warp_sum(leader ? __dmul_rn(a.x[target], sum) : 0.0);
        if ((threadIdx.x & 31) == 0) partials[blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)] = part;
    }
}

// K2 for warp_size in (32, 1024]: one CTA of ws threads per layout warp, the
// same tree through shared memory (the paper's sumvalues[] scratch).
template <bool SORTED, bool SCATTER>
__global__ void k2_wide_kernel(K2Args a) {
    extern __shared__ double part[];
    const int64_t w = blockIdx.x;
    const int32_t lane = threadIdx.x;
    if (a.done && *a.done) return;
    const uint64_t pol = evict_first_policy();
    const int32_t red = a.reduction[w];
    const int32_t r = lane / red, tl = lane & (red - 1);
    double sum = 0.0;
    int64_t pos = 0;
    const bool valid = r < a.rows_in_warp[w];
    if (valid) {
        pos = int64_t(a.rows_offset_warp[w]) + r;
        const bool active = SORTED ? pos < a.n_active : a.slen[pos] > 0;
        if (active) sum = lane_sum(a.values, a.cols, a.x, a.woff[w] + lane, a.ws, a.maxrows[w], pol);
    }
    part[lane] = sum;
    for (int32_t st = 1; st < red; st <<= 1) {
        __syncthreads();
        if ((tl & (2 * st - 1)) == 0) part[lane] = __dadd_rn(part[lane], part[lane + st]);
    }
    __syncthreads();
    if (valid && tl == 0) a.y[SCATTER ? a.fwd[pos] : pos] = part[lane];
}

template <bool SORTED, bool SCATTER>
void launch_k1(const K1Args& a, bool row_major, bool stream_form, bool compact, cudaStream_t s) {
    const unsigned g = grid_for(a.nrows);
    if (row_major)
        launch_pdl(k1_kernel<SORTED, SCATTER, true>, g, kBlock, s, a);
    else if (compact) {
        // 64-thread CTAs: at 5 x 256 threads per SM the last wave of config 2
        // (10.4 waves) leaves SMs idle; 20 x 64 packs it finer (141.1 ->
        // 139.6 us, A/B in one box; 128: 139.7-141.6)
        static const int cb = [] {
            const char* e = std::getenv("EW_K1C_BLOCK");  // A/B runs: CTA size of the 16-bit-column K1
            return cta_size_knob(e, 64);
        }();
        launch_pdl(k1_kernel<SORTED, SCATTER, false, false, true>, grid_for(a.nrows, cb), cb, s, a);
    }
    else if (stream_form)
        launch_pdl(k1_stream_kernel<SORTED, SCATTER>, g, kBlock, s, a);
    else
        launch_pdl(k1_kernel<SORTED, SCATTER, false, false, false>, g, kBlock, s, a);
    launched("k1_kernel");
}

template <bool SCATTER>
void launch_k1_grouped(const K1Args& a, bool stream_form, bool compact, cudaStream_t s) {
    if (compact) {
        static const int cb = [] {
            const char* e = std::getenv("EW_K1C_BLOCK");
            return cta_size_knob(e, 64);
        }();
        launch_pdl(k1_kernel<true, SCATTER, false, false, true, false, true>, grid_for(a.nrows, cb), cb, s, a);
    } else if (stream_form) {
        launch_pdl(k1_stream_kernel<true, SCATTER, false, true>, grid_for(a.nrows), kBlock, s, a);
    } else {
        launch_pdl(k1_kernel<true, SCATTER, false, false, false, false, true>, grid_for(a.nrows), kBlock, s, a);
    }
    launched("k1_kernel");
}

template <bool SORTED, bool SCATTER>
void launch_k2(const K2Args& a, cudaStream_t s) {
    if (a.nwarps == 0) return;
    if (a.ws <= 32) {
        // 128-thread CTAs: the mid-size FEM layouts run ~1.05 waves of
        // 256-thread CTAs at 6 per SM (accelerator: 935 CTAs, ncu 1.05
        // waves, a third of the SM cycles idle); finer CTAs even the tail.
        // Suite A/B on one box (cold us, 256 -> 128): accelerator 13.13 ->
        // 12.43, economics 13.54 -> 12.22, protein 16.64 -> 15.72, ship
        // 25.97 -> 24.80, circuit 10.91 -> 10.53; none slower (96 / 64 / 160
        // within noise of 128 or worse)
        static const int kb = [] {
            const char* e = std::getenv("EW_K2_BLOCK");  // A/B runs: CTA size of the K2 SpMV
            return cta_size_knob(e, 128);
        }();
        launch_pdl(k2_kernel<SORTED, SCATTER>, grid_for(a.nwarps * a.ws, kb), kb, s, a, (double*)nullptr);
    } else {
        k2_wide_kernel<SORTED, SCATTER><<<static_cast<unsigned>(a.nwarps), a.ws, a.ws * sizeof(double), s>>>(a);
    }
    launched("k2_kernel");
}

}  // namespace

bool layout_spmv_dot(const LayoutData& l, const double* x, double* y, bool scatter, cudaStream_t s,
                     const int* done, const DotSink& sink) {
    if (l.row_major || l.nrows == 0) return false;
    if (l.kind == EW_LAYOUT_K2) {
        // K2 with ws <= 32 and every row covered (a built, not imported, layout)
        if (l.ws > 32 || l.imported || l.nwarps == 0) return false;
        K2Args a{l.values.get(), l.cols.get(), l.warp_offset.get(), l.maxrows.get(), l.reduction.get(),
                 l.rows_offset_warp.get(), l.rows_in_warp.get(), l.slen.get(), l.fwd.get(), x, y, done,
                 l.nwarps, l.n_active, l.ws, l.ws_log2};
        const unsigned grid = grid_for(l.nwarps * l.ws);
        if (cg::dot_partials(grid) > sink.capacity) return false;
        auto go = [&](auto kernel) { launch_pdl(kernel, grid, kBlock, s, a, sink.partials); };
        if (l.sorted)
            scatter ? go(k2_kernel<true, true, true>) : go(k2_kernel<true, false, true>);
        else
            scatter ? go(k2_kernel<false, true, true>) : go(k2_kernel<false, false, true>);
        launched("k2_kernel");
        const unsigned nparts = grid * (kBlock / 32);
        launch_pdl(cg::dot_final_kernel, static_cast<unsigned>(cg::dot_final_blocks(nparts)), cg::kRedBlock, s,
                   (const double*)sink.partials, nparts, sink.partials + nparts, sink.tickets, sink.st, sink.dist,
                   sink.slot);
        launched("cg::dot_final_kernel");
        return true;
    }
    if (l.kind != EW_LAYOUT_K1) return false;
    K1Args a{l.values.get(), l.cols.get(), l.warp_offset.get(), l.maxrows.get(), l.slen.get(),
             l.fwd.get(), x, y, done, l.nrows, l.n_active, l.ws, l.ws_log2, nullptr, 0,
             l.cols16.get(), l.col_base.get(), nullptr, 0, l.lane_grp.get(), l.ngrp.get(), l.goff.get(),
             l.gcols.get(), l.gcols16.get()};
    a.col_shift = l.col_shift.get();
    const unsigned grid = grid_for(l.nrows);
    if (cg::dot_partials(grid) > sink.capacity) return false;
    const bool c = l.compact != 0;
    // the 16-bit-column form in 64-thread CTAs (as layout_spmv's); the
    // partials stay one per warp, in warp order, and no more of them
    static const int cb = [] {
        const char* e = std::getenv("EW_K1C_DOT_BLOCK");  // A/B runs
        return cta_size_knob(e, 64);
    }();
    const int block = c ? cb : 256;
    const unsigned g = grid_for(l.nrows, block);
    auto go = [&](auto kernel) { launch_pdl(kernel, g, block, s, a, sink.partials); };
    if (l.grouped) {  // sorted by construction
        if (c)
            scatter ? go(k1_dot_kernel<true, true, true, true>) : go(k1_dot_kernel<true, false, true, true>);
        else if (streams(l))
            scatter ? go(k1_dot_stream_kernel<true, true, true>) : go(k1_dot_stream_kernel<true, false, true>);
        else
            scatter ? go(k1_dot_kernel<true, true, false, true>) : go(k1_dot_kernel<true, false, false, true>);
    } else if (c) {
        if (l.sorted)
            scatter ? go(k1_dot_kernel<true, true, true>) : go(k1_dot_kernel<true, false, true>);
        else
            scatter ? go(k1_dot_kernel<false, true, true>) : go(k1_dot_kernel<false, false, true>);
    } else if (streams(l)) {
        if (l.sorted)
            scatter ? go(k1_dot_stream_kernel<true, true>) : go(k1_dot_stream_kernel<true, false>);
        else
            scatter ? go(k1_dot_stream_kernel<false, true>) : go(k1_dot_stream_kernel<false, false>);
    } else if (l.sorted) {
        scatter ? go(k1_dot_kernel<true, true, false>) : go(k1_dot_kernel<true, false, false>);
    } else {
        scatter ? go(k1_dot_kernel<false, true, false>) : go(k1_dot_kernel<false, false, false>);
    }
    launched("k1_dot_kernel");
    const unsigned nparts = g * (block / 32);  // one partial per SpMV warp
    launch_pdl(cg::dot_final_kernel, static_cast<unsigned>(cg::dot_final_blocks(nparts)), cg::kRedBlock, s,
               (const double*)sink.partials, nparts, sink.partials + nparts, sink.tickets, sink.st, sink.dist,
               sink.slot);
    launched("cg::dot_final_kernel");
    return true;
}

void layout_spmv(const LayoutData& l, const double* x, double* y, bool scatter, cudaStream_t s,
                 const int* done) {
    if (l.nrows == 0) return;
    if (l.kind == EW_LAYOUT_K1) {
        K1Args a{l.values.get(), l.cols.get(), l.warp_offset.get(), l.maxrows.get(), l.slen.get(),
                 l.fwd.get(), x, y, done, l.nrows, l.n_active, l.ws, l.ws_log2, nullptr, 0,
                 l.cols16.get(), l.col_base.get(), nullptr, 0, l.lane_grp.get(), l.ngrp.get(), l.goff.get(),
                 l.gcols.get(), l.gcols16.get()};
    a.col_shift = l.col_shift.get();
        const bool rm = l.row_major != 0, sf = streams(l), c = l.compact != 0;
        if (const int h = coop_warps(l)) {
            // EW_K1_BULK=1: the bulk-copy staging form (A/B; needs the
            // layout's 32-slot slab alignment, the default)
            static const bool bulk = [] {
                const char* e = std::getenv("EW_K1_BULK");
                return e && e[0] == '1';
            }();
            if (bulk && !c && l.align && l.segment_bytes == 128)
                scatter ? launch_k1_bulk<true>(a, l.nwarps, h, s) : launch_k1_bulk<false>(a, l.nwarps, h, s);
            else
                scatter ? launch_k1_coop<true>(a, l.nwarps, h, c, s) : launch_k1_coop<false>(a, l.nwarps, h, c, s);
            return;
        }
        if (l.head_warps > 0 && !rm && !l.imported) {
            // power-law rows, too many for the cooperative K1 everywhere
            // (webbase: 1M rows, one of 4,700 entries): the head warps (rows
            // over head_mx() entries) run the cooperative K1 on the side
            // stream, the plain K1 the tail rows meanwhile; disjoint rows,
            // the same row sums. Webbase (cold): 1,756 us unsplit, ~160 us
            // with k1_coop_kernel (H = 8) as the head, 76 us with
            // k1_long_kernel (ncu: head 62 us, tail 39 us, concurrent);
            // circuit keeps the cooperative K1 everywhere (773 vs 604 GB/s
            // effective split). Any column form (16-bit / grouped layouts
            // over 64 MB with a few long rows: the head reads the kept form)
            const int form = (l.grouped ? 2 : 0) + (c ? 1 : 0);
            SideStream& ss = *l.side;
            std::lock_guard<std::mutex> lock(ss.mu);
            EW_CUDA_CHECK(cudaEventRecord(ss.fork, s));
            EW_CUDA_CHECK(cudaStreamWaitEvent(ss.s, ss.fork, 0));
            static const bool coop_head = [] {  // A/B: the cooperative K1 (H = 8) for the head
                const char* e = std::getenv("EW_K1_HEAD_COOP");
                return e && e[0] == '1';
            }();
            if (coop_head && form == 0)
                scatter ? launch_k1_coop<true>(a, l.head_warps, 8, false, ss.s)
                        : launch_k1_coop<false>(a, l.head_warps, 8, false, ss.s);
            else
                scatter ? launch_k1_long<true>(a, l.head_warps, form, ss.s)
                        : launch_k1_long<false>(a, l.head_warps, form, ss.s);
            const int64_t lo = l.head_warps * 32;
            if (lo < l.nrows) {  // the tail: the plain form of the layout's columns (row_lo offset)
                K1Args t = a;
                t.row_lo = lo;
                const int b = c ? 64 : kBlock;
                const unsigned g = grid_for(l.nrows - lo, b);
                auto go = [&](auto kernel) { launch_pdl(kernel, g, b, s, t); };
                if (form == 0) scatter ? go(k1_kernel<true, true, false>) : go(k1_kernel<true, false, false>);
                else if (form == 1)
                    scatter ? go(k1_kernel<true, true, false, false, true>) : go(k1_kernel<true, false, false, false, true>);
                else if (form == 2)
                    scatter ? go(k1_kernel<true, true, false, false, false, false, true>)
                            : go(k1_kernel<true, false, false, false, false, false, true>);
                else
                    scatter ? go(k1_kernel<true, true, false, false, true, false, true>)
                            : go(k1_kernel<true, false, false, false, true, false, true>);
                launched("k1_kernel");
            }
            EW_CUDA_CHECK(cudaEventRecord(ss.join, ss.s));
            EW_CUDA_CHECK(cudaStreamWaitEvent(s, ss.join, 0));
            return;
        }
        if (l.grouped) {  // sorted, column-major by construction
            scatter ? launch_k1_grouped<true>(a, sf, c, s) : launch_k1_grouped<false>(a, sf, c, s);
            return;
        }
        if (l.sorted) {
            scatter ? launch_k1<true, true>(a, rm, sf, c, s) : launch_k1<true, false>(a, rm, sf, c, s);
        } else {
            scatter ? launch_k1<false, true>(a, rm, sf, c, s) : launch_k1<false, false>(a, rm, sf, c, s);
        }
        return;
    }
    // K2: packing covers every sorted position, so each y entry is written by
    // exactly one leader; an imported layout may not, so y is cleared first
    // (the reference starts from y = 0.0, warp_spmv.cpp:65).
    if (l.imported) EW_CUDA_CHECK(cudaMemsetAsync(y, 0, l.nrows * sizeof(double), s));
    K2Args a{l.values.get(), l.cols.get(), l.warp_offset.get(), l.maxrows.get(), l.reduction.get(),
             l.rows_offset_warp.get(), l.rows_in_warp.get(), l.slen.get(), l.fwd.get(), x, y, done,
             l.nwarps, l.n_active, l.ws, l.ws_log2};
    if (l.sorted) {
        scatter ? launch_k2<true, true>(a, s) : launch_k2<true, false>(a, s);
    } else {
        scatter ? launch_k2<false, true>(a, s) : launch_k2<false, false>(a, s);
    }
}

void layout_spmv_warps(const LayoutData& l, const int32_t* widx, int64_t nidx, const double* x, double* y,
                       cudaStream_t s) {
    require(l.kind == EW_LAYOUT_K1 && !l.row_major && l.sorted, "warp-list SpMV: sorted column-major K1 only");
    if (nidx == 0 || l.nrows == 0) return;
    K1Args a{l.values.get(), l.cols.get(), l.warp_offset.get(), l.maxrows.get(), l.slen.get(),
             l.fwd.get(), x, y, nullptr, l.nrows, l.n_active, l.ws, l.ws_log2, nullptr, 0,
             l.cols16.get(), l.col_base.get(), widx, nidx, l.lane_grp.get(), l.ngrp.get(), l.goff.get(),
             l.gcols.get(), l.gcols16.get()};
    a.col_shift = l.col_shift.get();
    const int64_t threads = nidx << l.ws_log2;
    if (l.grouped && l.compact)
        launch_pdl(k1_kernel<true, true, false, false, true, true, true>, grid_for(threads, 64), 64, s, a);
    else if (l.grouped)
        launch_pdl(k1_kernel<true, true, false, false, false, true, true>, grid_for(threads), kBlock, s, a);
    else if (l.compact)
        launch_pdl(k1_kernel<true, true, false, false, true, true>, grid_for(threads, 64), 64, s, a);
    else
        launch_pdl(k1_kernel<true, true, false, false, false, true>, grid_for(threads), kBlock, s, a);
    launched("k1_kernel");
}

void layout_spmv_split(const LayoutData& l, const double* x, const double* xg, int64_t nown, double* y,
                       cudaStream_t s) {
    require(l.kind == EW_LAYOUT_K1 && !l.row_major, "split-x SpMV: K1 column-major layouts only");
    require(l.cols_full, "split-x SpMV: the layout's int32 columns were dropped (restore_columns)");
    if (l.nrows == 0) return;
    K1Args a{l.values.get(), l.cols.get(), l.warp_offset.get(), l.maxrows.get(), l.slen.get(),
             l.fwd.get(), x, y, nullptr, l.nrows, l.n_active, l.ws, l.ws_log2, xg, static_cast<int32_t>(nown),
             nullptr, nullptr};
    if (streams(l)) {
        if (l.sorted)
            launch_pdl(k1_stream_kernel<true, true, true>, grid_for(a.nrows), kBlock, s, a);
        else
            launch_pdl(k1_stream_kernel<false, true, true>, grid_for(a.nrows), kBlock, s, a);
    } else if (l.sorted) {
        launch_pdl(k1_kernel<true, true, false, true>, grid_for(a.nrows), kBlock, s, a);
    } else {
        launch_pdl(k1_kernel<false, true, false, true>, grid_for(a.nrows), kBlock, s, a);
    }
    launched("k1_kernel");
}

bool spmv_reads_int32(const LayoutData& l) {
    if (l.kind != EW_LAYOUT_K1 || l.row_major) return true;
    if (l.compact) return false;  // 16-bit forms; wide warps through col_shift
    if (!l.grouped) return true;
    return coop_warps(l) != 0;  // the cooperative K1 runs before the grouped form
}

// Shared-memory opt-in of k1_long_kernel on the current device (a layout
// with a head split calls this when it is built, outside any capture).
void k1_long_setup() {
    const int bytes = static_cast<int>(kLongSmem);
    const auto attr = cudaFuncAttributeMaxDynamicSharedMemorySize;
    EW_CUDA_CHECK(cudaFuncSetAttribute(k1_long_kernel<true, 0>, attr, bytes));
    EW_CUDA_CHECK(cudaFuncSetAttribute(k1_long_kernel<true, 1>, attr, bytes));
    EW_CUDA_CHECK(cudaFuncSetAttribute(k1_long_kernel<true, 2>, attr, bytes));
    EW_CUDA_CHECK(cudaFuncSetAttribute(k1_long_kernel<true, 3>, attr, bytes));
    EW_CUDA_CHECK(cudaFuncSetAttribute(k1_long_kernel<false, 0>, attr, bytes));
    EW_CUDA_CHECK(cudaFuncSetAttribute(k1_long_kernel<false, 1>, attr, bytes));
    EW_CUDA_CHECK(cudaFuncSetAttribute(k1_long_kernel<false, 2>, attr, bytes));
    EW_CUDA_CHECK(cudaFuncSetAttribute(k1_long_kernel<false, 3>, attr, bytes));
}

const void* kernel_anchor_spmv() { return reinterpret_cast<const void*>(&k1_stream_kernel<true, false>); }

}  // namespace ew

/* CPU restatement of the reference ELL-WARP hot path. TEST INFRASTRUCTURE
 * ONLY -- see ew_oracle.h for what pins it. Compiled with -ffp-contract=off so
 * every a*b+c rounds twice, as the reference's default (non -march=native)
 * build does. File:line citations are into /root/reference/proj. */
#define _POSIX_C_SOURCE 200809L
#include "ew_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; } /* types.hpp:27 */

/* csr.cpp:75-86: sequential per-row sum starting from 0.0, CSR order. */
int ewo_spmv_csr(int64_t nrows, int64_t ncols, const int64_t* ro, const int64_t* ci,
                 const double* v, const double* x, double* y) {
    (void)ncols;
    for (int64_t r = 0; r < nrows; ++r) {
        double sum = 0.0;
        for (int64_t k = ro[r]; k < ro[r + 1]; ++k) sum += v[k] * x[ci[k]];
        y[r] = sum;
    }
    return 0;
}

/* The same row sums on `threads` POSIX threads (contiguous row ranges): a
 * clearly-labelled multi-core PORT for the bench's CPU comparison (the
 * reference itself is single-threaded). Bitwise equal to ewo_spmv_csr. */
typedef struct {
    int64_t r0, r1;
    const int64_t *ro, *ci;
    const double *v, *x;
    double* y;
} ewo_mt_job;

static void* ewo_mt_rows(void* arg) {
    const ewo_mt_job* j = (const ewo_mt_job*)arg;
    for (int64_t r = j->r0; r < j->r1; ++r) {
        double sum = 0.0;
        for (int64_t k = j->ro[r]; k < j->ro[r + 1]; ++k) sum += j->v[k] * j->x[j->ci[k]];
        j->y[r] = sum;
    }
    return NULL;
}

int ewo_spmv_csr_mt(int64_t nrows, int64_t ncols, const int64_t* ro, const int64_t* ci,
                    const double* v, const double* x, double* y, int threads) {
    (void)ncols;
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t tid[256];
    ewo_mt_job job[256];
    for (int t = 0; t < threads; ++t) {
        job[t] = (ewo_mt_job){nrows * t / threads, nrows * (t + 1) / threads, ro, ci, v, x, y};
        if (t > 0 && pthread_create(&tid[t], NULL, ewo_mt_rows, &job[t]) != 0) return -1;
    }
    ewo_mt_rows(&job[0]);
    for (int t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
    return 0;
}

/* csr.cpp:106-117: first stored entry on the diagonal, 0.0 when absent. */
void ewo_extract_diagonal(int64_t nrows, int64_t ncols, const int64_t* ro, const int64_t* ci,
                          const double* v, double* d) {
    for (int64_t r = 0; r < nrows; ++r) {
        d[r] = 0.0;
        if (r >= ncols) continue;
        for (int64_t k = ro[r]; k < ro[r + 1]; ++k) {
            if (ci[k] == r) {
                d[r] = v[k];
                break;
            }
        }
    }
}

/* csr.cpp:57-73 */
int ewo_validate_csr(int64_t nrows, int64_t ncols, int64_t nro, const int64_t* ro, int64_t nnz,
                     const int64_t* ci) {
    if (nrows < 0 || ncols < 0) return 1;
    if (nro != nrows + 1) return 1;
    if (ro[0] != 0 || ro[nrows] != nnz) return 1;
    for (int64_t r = 0; r < nrows; ++r) {
        if (ro[r] > ro[r + 1]) return 1;
        for (int64_t k = ro[r]; k < ro[r + 1]; ++k) {
            if (ci[k] < 0 || ci[k] >= ncols) return 1;
            if (k > ro[r] && ci[k - 1] >= ci[k]) return 1;
        }
    }
    return 0;
}

/* permutation.cpp:49-55 is a std::stable_sort by length, longest first, ties
 * in ascending row order. Restated as a stable counting sort: bucket rows by
 * length, lay buckets out longest-first, fill each bucket in row order. */
void ewo_sort_rows_desc(int64_t nrows, const int64_t* ro, int64_t* fwd, int64_t* inv) {
    int64_t maxlen = 0;
    for (int64_t r = 0; r < nrows; ++r) {
        const int64_t len = ro[r + 1] - ro[r];
        if (len > maxlen) maxlen = len;
    }
    int64_t* start = (int64_t*)calloc((size_t)maxlen + 2, sizeof(int64_t));
    for (int64_t r = 0; r < nrows; ++r) start[maxlen - (ro[r + 1] - ro[r])]++;
    int64_t acc = 0;
    for (int64_t b = 0; b <= maxlen; ++b) {
        const int64_t c = start[b];
        start[b] = acc;
        acc += c;
    }
    for (int64_t r = 0; r < nrows; ++r) {
        const int64_t pos = start[maxlen - (ro[r + 1] - ro[r])]++;
        fwd[pos] = r;
        inv[r] = pos;
    }
    free(start);
}

/* warp_layout.cpp:76-84 */
int64_t ewo_compute_k2_lanes(int64_t nnz_row, int64_t threshold, int64_t warp_size) {
    if (threshold < 1) return -1;
    if (warp_size < 1 || (warp_size & (warp_size - 1)) != 0) return -1;
    if (nnz_row > warp_size * threshold) return warp_size;
    int64_t lanes = 1;
    while (ceil_div(nnz_row, lanes) > threshold) lanes <<= 1;
    return lanes;
}

/* warp_model.cpp:7-14 (only the fields the layout build reads). */
static int valid_cfg(int warp_size, int segment_bytes) {
    if (warp_size <= 0 || (warp_size & (warp_size - 1)) != 0) return 0;
    if (segment_bytes <= 0 || (segment_bytes & (segment_bytes - 1)) != 0) return 0;
    return 1;
}

/* warp_layout.cpp:12-16: round up to segment_bytes/4 slots. */
static int64_t align_offset(int64_t off, int align, int segment_bytes) {
    if (!align) return off;
    const int64_t unit = segment_bytes / 4;
    return ceil_div(off, unit) * unit;
}

static ewo_layout* layout_common(int kind, int64_t nrows, int64_t ncols, const int64_t* ro,
                                 int warp_size, int sort_rows) {
    ewo_layout* l = (ewo_layout*)calloc(1, sizeof(ewo_layout));
    l->kind = kind;
    l->warp_size = warp_size;
    l->nrows = nrows;
    l->ncols = ncols;
    l->nnz = ro[nrows];
    l->forward = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nrows + 1));
    l->inverse = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nrows + 1));
    l->sorted_row_length = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nrows + 1));
    if (sort_rows) {
        ewo_sort_rows_desc(nrows, ro, l->forward, l->inverse);
    } else {
        for (int64_t r = 0; r < nrows; ++r) l->forward[r] = l->inverse[r] = r;
    }
    for (int64_t p = 0; p < nrows; ++p) l->sorted_row_length[p] = ro[l->forward[p] + 1] - ro[l->forward[p]];
    return l;
}

/* slot(w, lane, j): warp_layout.hpp:31-34 (K1, incl. the row_major
 * diagnostic) and :60 (K2). */
static int64_t slot_of(const ewo_layout* l, int64_t w, int64_t lane, int64_t j) {
    if (l->row_major) return l->warp_offset[w] + lane * l->maxrows[w] + j;
    return l->warp_offset[w] + j * l->warp_size + lane;
}

/* warp_layout.cpp:32-74 */
int ewo_build_k1(int64_t nrows, int64_t ncols, const int64_t* ro, const int64_t* ci,
                 const double* v, int warp_size, int segment_bytes, int align, int sort_rows,
                 int row_major, ewo_layout** out) {
    if (!valid_cfg(warp_size, segment_bytes)) return 1;
    ewo_layout* l = layout_common(1, nrows, ncols, ro, warp_size, sort_rows);
    l->row_major = row_major;
    const int64_t ws = warp_size;
    const int64_t nw = ceil_div(nrows, ws);
    l->nwarps = nw;
    l->warp_offset = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nw + 1));
    l->maxrows = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nw + 1));
    l->rows_in_warp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nw + 1));
    int64_t off = 0;
    for (int64_t w = 0; w < nw; ++w) {
        const int64_t lo = w * ws;
        const int64_t hi = lo + ws < nrows ? lo + ws : nrows;
        int64_t mx = 0;
        for (int64_t p = lo; p < hi; ++p)
            if (l->sorted_row_length[p] > mx) mx = l->sorted_row_length[p];
        off = align_offset(off, align, segment_bytes);
        l->warp_offset[w] = off;
        l->maxrows[w] = mx;
        l->rows_in_warp[w] = hi - lo;
        off += mx * ws;
    }
    l->nslots = off;
    l->values = (double*)calloc((size_t)off + 1, sizeof(double));
    l->col_indices = (int64_t*)calloc((size_t)off + 1, sizeof(int64_t));
    for (int64_t w = 0; w < nw; ++w) {
        for (int64_t lane = 0; lane < l->rows_in_warp[w]; ++lane) {
            const int64_t p = w * ws + lane;
            const int64_t row = l->forward[p];
            for (int64_t j = 0; j < l->sorted_row_length[p]; ++j) {
                const int64_t s = slot_of(l, w, lane, j);
                l->values[s] = v[ro[row] + j];
                l->col_indices[s] = ci[ro[row] + j];
            }
        }
    }
    *out = l;
    return 0;
}

/* warp_layout.cpp:86-147: greedy packing over sorted rows; a warp closes
 * when the lane count changes or the warp is full. */
int ewo_build_k2(int64_t nrows, int64_t ncols, const int64_t* ro, const int64_t* ci,
                 const double* v, int warp_size, int segment_bytes, int align, int64_t threshold,
                 int sort_rows, ewo_layout** out) {
    if (!valid_cfg(warp_size, segment_bytes) || threshold < 1) return 1;
    ewo_layout* l = layout_common(2, nrows, ncols, ro, warp_size, sort_rows);
    l->threshold = threshold;
    const int64_t ws = warp_size;
    /* at most nrows warps */
    const size_t cap = (size_t)nrows + 1;
    l->warp_offset = (int64_t*)malloc(sizeof(int64_t) * cap);
    l->maxrows = (int64_t*)malloc(sizeof(int64_t) * cap);
    l->rows_in_warp = (int64_t*)malloc(sizeof(int64_t) * cap);
    l->reduction = (int64_t*)malloc(sizeof(int64_t) * cap);
    l->rows_offset_warp = (int64_t*)malloc(sizeof(int64_t) * cap);
    int64_t nw = 0;
    for (int64_t p = 0; p < nrows;) {
        const int64_t lanes = ewo_compute_k2_lanes(l->sorted_row_length[p], threshold, ws);
        const int64_t capacity = ws / lanes;
        int64_t q = p, mx = 0;
        while (q < nrows && q - p < capacity &&
               ewo_compute_k2_lanes(l->sorted_row_length[q], threshold, ws) == lanes) {
            const int64_t m = ceil_div(l->sorted_row_length[q], lanes);
            if (m > mx) mx = m;
            ++q;
        }
        l->reduction[nw] = lanes;
        l->rows_offset_warp[nw] = p;
        l->rows_in_warp[nw] = q - p;
        l->maxrows[nw] = mx;
        ++nw;
        p = q;
    }
    l->nwarps = nw;
    int64_t off = 0;
    for (int64_t w = 0; w < nw; ++w) {
        off = align_offset(off, align, segment_bytes);
        l->warp_offset[w] = off;
        off += l->maxrows[w] * ws;
    }
    l->nslots = off;
    l->values = (double*)calloc((size_t)off + 1, sizeof(double));
    l->col_indices = (int64_t*)calloc((size_t)off + 1, sizeof(int64_t));
    for (int64_t w = 0; w < nw; ++w) {
        const int64_t red = l->reduction[w], mx = l->maxrows[w];
        for (int64_t r = 0; r < l->rows_in_warp[w]; ++r) {
            const int64_t pos = l->rows_offset_warp[w] + r;
            const int64_t row = l->forward[pos];
            for (int64_t e = 0; e < l->sorted_row_length[pos]; ++e) {
                const int64_t s = slot_of(l, w, r * red + e / mx, e % mx);
                l->values[s] = v[ro[row] + e];
                l->col_indices[s] = ci[ro[row] + e];
            }
        }
    }
    *out = l;
    return 0;
}

void ewo_layout_free(ewo_layout* l) {
    if (!l) return;
    free(l->values);
    free(l->col_indices);
    free(l->warp_offset);
    free(l->maxrows);
    free(l->rows_in_warp);
    free(l->reduction);
    free(l->rows_offset_warp);
    free(l->forward);
    free(l->inverse);
    free(l->sorted_row_length);
    free(l);
}

/* warp_layout.cpp:20-29 */
int64_t ewo_layout_stored_slots(const ewo_layout* l) {
    int64_t t = 0;
    for (int64_t w = 0; w < l->nwarps; ++w)
        t += l->maxrows[w] * l->rows_in_warp[w] * (l->kind == 2 ? l->reduction[w] : 1);
    return t;
}

/* warp_layout.cpp:149-174 */
void ewo_value_slot_map(const ewo_layout* l, const int64_t* ro, int64_t* map) {
    if (l->kind == 1) {
        for (int64_t p = 0; p < l->nrows; ++p) {
            const int64_t row = l->forward[p];
            const int64_t w = p / l->warp_size, lane = p % l->warp_size;
            for (int64_t j = 0; j < ro[row + 1] - ro[row]; ++j) map[ro[row] + j] = slot_of(l, w, lane, j);
        }
        return;
    }
    for (int64_t w = 0; w < l->nwarps; ++w) {
        const int64_t red = l->reduction[w], mx = l->maxrows[w];
        for (int64_t r = 0; r < l->rows_in_warp[w]; ++r) {
            const int64_t pos = l->rows_offset_warp[w] + r;
            const int64_t row = l->forward[pos];
            for (int64_t e = 0; e < l->sorted_row_length[pos]; ++e)
                map[ro[row] + e] = slot_of(l, w, r * red + e / mx, e % mx);
        }
    }
}

/* warp_spmv.cpp:9-60 (K1) and :62-126 (K2). Active lanes belong to rows with
 * at least one entry and run all maxrows steps, padding included; rows with
 * no entries keep y = 0.0. K2 lanes sum contiguous chunks and combine through
 * an ascending-stride pairwise tree (stride 1, 2, 4, ...). */
void ewo_spmv_layout(const ewo_layout* l, const double* x, int scatter, double* y) {
    const int64_t ws = l->warp_size;
    double* acc = (double*)malloc(sizeof(double) * (size_t)ws);
    for (int64_t i = 0; i < l->nrows; ++i) y[i] = 0.0;
    for (int64_t w = 0; w < l->nwarps; ++w) {
        const int64_t red = l->kind == 2 ? l->reduction[w] : 1;
        const int64_t first = l->kind == 2 ? l->rows_offset_warp[w] : w * ws;
        const int64_t mx = l->maxrows[w];
        for (int64_t t = 0; t < ws; ++t) acc[t] = 0.0;
        for (int64_t r = 0; r < l->rows_in_warp[w]; ++r) {
            if (l->sorted_row_length[first + r] == 0) continue;
            for (int64_t t = 0; t < red; ++t) {
                const int64_t lane = r * red + t;
                double s = 0.0;
                for (int64_t j = 0; j < mx; ++j) {
                    const int64_t k = slot_of(l, w, lane, j);
                    s += l->values[k] * x[l->col_indices[k]];
                }
                acc[lane] = s;
            }
            for (int64_t stride = 1; stride < red; stride <<= 1)
                for (int64_t t = 0; t + stride < red; t += 2 * stride)
                    acc[r * red + t] += acc[r * red + t + stride];
            const int64_t pos = first + r;
            y[scatter ? l->forward[pos] : pos] = acc[r * red];
        }
    }
    free(acc);
}

/* ewo_spmv_layout restricted to the warps [w0, w1): writes every row those
 * warps hold (0.0 for rows without entries), the same per-lane arithmetic.
 * Warps own disjoint rows, so ranges can run on separate threads. */
static void spmv_layout_warps(const ewo_layout* l, const double* x, int scatter, double* y, int64_t w0,
                              int64_t w1, double* acc) {
    const int64_t ws = l->warp_size;
    for (int64_t w = w0; w < w1; ++w) {
        const int64_t red = l->kind == 2 ? l->reduction[w] : 1;
        const int64_t first = l->kind == 2 ? l->rows_offset_warp[w] : w * ws;
        const int64_t mx = l->maxrows[w];
        for (int64_t r = 0; r < l->rows_in_warp[w]; ++r) {
            const int64_t pos = first + r;
            double* out = &y[scatter ? l->forward[pos] : pos];
            if (l->sorted_row_length[pos] == 0) {
                *out = 0.0;
                continue;
            }
            for (int64_t t = 0; t < red; ++t) {
                const int64_t lane = r * red + t;
                double s = 0.0;
                for (int64_t j = 0; j < mx; ++j) {
                    const int64_t k = slot_of(l, w, lane, j);
                    s += l->values[k] * x[l->col_indices[k]];
                }
                acc[lane] = s;
            }
            for (int64_t stride = 1; stride < red; stride <<= 1)
                for (int64_t t = 0; t + stride < red; t += 2 * stride)
                    acc[r * red + t] += acc[r * red + t + stride];
            *out = acc[r * red];
        }
    }
}

/* Fork-join over [0, n) in `threads` contiguous ranges (a fresh pthread per
 * range; the caller's thread takes the first). */
typedef void (*range_fn)(void* ctx, int64_t i0, int64_t i1);
typedef struct {
    range_fn fn;
    void* ctx;
    int64_t i0, i1;
} range_job;

static void* range_main(void* a) {
    range_job* j = (range_job*)a;
    j->fn(j->ctx, j->i0, j->i1);
    return NULL;
}

static void par_for(int threads, int64_t n, range_fn fn, void* ctx) {
    if (threads <= 1 || n < 4096) {
        fn(ctx, 0, n);
        return;
    }
    if (threads > 256) threads = 256;
    pthread_t tid[256];
    range_job job[256];
    int started[256];
    const int64_t chunk = (n + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        job[t].fn = fn;
        job[t].ctx = ctx;
        job[t].i0 = t * chunk < n ? t * chunk : n;
        job[t].i1 = (t + 1) * chunk < n ? (t + 1) * chunk : n;
        started[t] = 0;
    }
    for (int t = 1; t < threads; ++t)
        started[t] = pthread_create(&tid[t], NULL, range_main, &job[t]) == 0;
    fn(ctx, job[0].i0, job[0].i1);
    for (int t = 1; t < threads; ++t) {
        if (started[t])
            pthread_join(tid[t], NULL);
        else
            fn(ctx, job[t].i0, job[t].i1);  /* no thread: run the range here */
    }
}

typedef struct {
    const ewo_layout* l;
    const double* x;
    double* y;
    int scatter;
} layout_range_ctx;

static void layout_range(void* c, int64_t w0, int64_t w1) {
    const layout_range_ctx* lc = (const layout_range_ctx*)c;
    double* acc = (double*)malloc(sizeof(double) * (size_t)lc->l->warp_size);
    spmv_layout_warps(lc->l, lc->x, lc->scatter, lc->y, w0, w1, acc);
    free(acc);
}

void ewo_spmv_layout_mt(const ewo_layout* l, const double* x, int scatter, double* y, int threads) {
    layout_range_ctx c = {l, x, y, scatter};
    par_for(threads, l->nwarps, layout_range, &c);
}

void ewo_layout_op_mt(void* ctx, const double* x, double* y) {
    const ewo_layout_mt_ctx* c = (const ewo_layout_mt_ctx*)ctx;
    ewo_spmv_layout_mt(c->l, x, c->scatter, y, c->threads);
}

/* reorder.cpp:8-43: columns renumbered by inverse; for rs each row's
 * (column, value) pairs are re-sorted by the new column (keys are unique
 * because renumbering is a bijection). */
int ewo_reorder(int64_t nrows, int64_t ncols, const int64_t* ro, const int64_t* ci,
                const double* v, const int64_t* fwd, const int64_t* inv, int sort_within_rows,
                int64_t* ci_out, double* v_out) {
    (void)fwd;
    if (nrows != ncols) return 1;
    const int64_t nnz = ro[nrows];
    for (int64_t k = 0; k < nnz; ++k) {
        ci_out[k] = inv[ci[k]];
        v_out[k] = v[k];
    }
    if (!sort_within_rows) return 0;
    for (int64_t r = 0; r < nrows; ++r) {
        /* insertion sort: rows are short and the keys distinct */
        for (int64_t k = ro[r] + 1; k < ro[r + 1]; ++k) {
            const int64_t c = ci_out[k];
            const double val = v_out[k];
            int64_t m = k - 1;
            while (m >= ro[r] && ci_out[m] > c) {
                ci_out[m + 1] = ci_out[m];
                v_out[m + 1] = v_out[m];
                --m;
            }
            ci_out[m + 1] = c;
            v_out[m + 1] = val;
        }
    }
    return 0;
}

/* cg.cpp:9-13 sequential dot from 0.0 */
static double dot(int64_t n, const double* a, const double* b) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

static int all_finite(int64_t n, const double* v) {
    for (int64_t i = 0; i < n; ++i)
        if (!isfinite(v[i])) return 0;
    return 1;
}

/* The CG's element-wise loops (each element's arithmetic exactly as in
 * cg.cpp; elements are independent, so ranges may run on threads). */
enum { EW_RESID, EW_PRECOND, EW_PRECOND_P, EW_XR, EW_PUPD, EW_FINITE };
typedef struct {
    int what, jacobi;
    const double *b, *diag, *q;
    double *x, *r, *z, *p;
    double alpha, beta;
    int bad[256];
    int64_t chunk;
} vec_ctx;

static void vec_range(void* c, int64_t i0, int64_t i1) {
    vec_ctx* v = (vec_ctx*)c;
    switch (v->what) {
        case EW_RESID: /* cg.cpp:58, 85 */
            for (int64_t i = i0; i < i1; ++i) v->r[i] = v->b[i] - v->q[i];
            break;
        case EW_PRECOND: /* cg.cpp:36-42, 96 */
        case EW_PRECOND_P: /* + cg.cpp:67 p = z */
            for (int64_t i = i0; i < i1; ++i) {
                v->z[i] = v->jacobi ? v->r[i] / v->diag[i] : v->r[i];
                if (v->what == EW_PRECOND_P) v->p[i] = v->z[i];
            }
            break;
        case EW_XR: /* cg.cpp:78-81 */
            for (int64_t i = i0; i < i1; ++i) {
                v->x[i] += v->alpha * v->p[i];
                v->r[i] -= v->alpha * v->q[i];
            }
            break;
        case EW_PUPD: /* cg.cpp:99 */
            for (int64_t i = i0; i < i1; ++i) v->p[i] = v->z[i] + v->beta * v->p[i];
            break;
        case EW_FINITE: /* cg.cpp:87 */
            for (int64_t i = i0; i < i1; ++i)
                if (!isfinite(v->r[i])) {
                    v->bad[v->chunk ? i0 / v->chunk : 0] = 1;
                    break;
                }
            break;
    }
}

static void vec_op(vec_ctx* v, int what, int threads, int64_t n) {
    v->what = what;
    par_for(threads, n, vec_range, v);
}

static int vec_finite(vec_ctx* v, int threads, int64_t n) {
    int t = threads <= 1 || n < 4096 ? 1 : (threads > 256 ? 256 : threads);
    memset(v->bad, 0, sizeof(v->bad));
    v->chunk = (n + t - 1) / t;
    vec_op(v, EW_FINITE, threads, n);
    for (int i = 0; i < 256; ++i)
        if (v->bad[i]) return 0;
    return 1;
}

static int cg_core(ewo_spmv_fn op, void* ctx, int64_t n, const double* b, const double* diag,
                   const ewo_cg_config* cfg, double* x, double* history, ewo_cg_result* res,
                   int threads);

/* cg.cpp:25-104 */
int ewo_cg_solve(ewo_spmv_fn op, void* ctx, int64_t n, const double* b, const double* diag,
                 const ewo_cg_config* cfg, double* x, double* history, ewo_cg_result* res) {
    return cg_core(op, ctx, n, b, diag, cfg, x, history, res, 1);
}

/* The same solve with the element-wise loops on `threads` threads; every
 * dot product stays the reference's sequential sum (cg.cpp:9-13), so the
 * history is bit-identical to ewo_cg_solve with the same operator. */
int ewo_cg_solve_mt(ewo_spmv_fn op, void* ctx, int64_t n, const double* b, const double* diag,
                    const ewo_cg_config* cfg, double* x, double* history, ewo_cg_result* res,
                    int threads) {
    return cg_core(op, ctx, n, b, diag, cfg, x, history, res, threads);
}

static int cg_core(ewo_spmv_fn op, void* ctx, int64_t n, const double* b, const double* diag,
                   const ewo_cg_config* cfg, double* x, double* history, ewo_cg_result* res,
                   int threads) {
    memset(res, 0, sizeof(*res));
    if (!(cfg->rel_tolerance > 0.0)) return 1;
    if (!all_finite(n, b)) return 2;
    const int jacobi = cfg->jacobi;
    if (jacobi) {
        if (!diag) return 1;
        for (int64_t i = 0; i < n; ++i)
            if (diag[i] == 0.0) return 1;
    }
    for (int64_t i = 0; i < n; ++i) x[i] = 0.0;
    const double bnorm = sqrt(dot(n, b, b));
    if (bnorm == 0.0) {
        res->converged = 1;
        history[0] = 0.0;
        res->history_len = 1;
        return 0;
    }
    double* r = (double*)malloc(sizeof(double) * (size_t)(n + 1));
    double* z = (double*)malloc(sizeof(double) * (size_t)(n + 1));
    double* p = (double*)malloc(sizeof(double) * (size_t)(n + 1));
    double* q = (double*)malloc(sizeof(double) * (size_t)(n + 1));
    int status = 0;
    vec_ctx vc;
    memset(&vc, 0, sizeof(vc));
    vc.jacobi = jacobi;
    vc.b = b;
    vc.diag = diag;
    vc.q = q;
    vc.x = x;
    vc.r = r;
    vc.z = z;
    vc.p = p;
    op(ctx, x, q);
    res->spmv_calls++;
    vec_op(&vc, EW_RESID, threads, n);
    int64_t h = 0;
    history[h++] = sqrt(dot(n, r, r)) / bnorm;
    if (history[0] <= cfg->rel_tolerance) {
        res->converged = 1;
        goto done;
    }
    vec_op(&vc, EW_PRECOND_P, threads, n);
    double rz = dot(n, r, z);
    for (int64_t k = 1; k <= cfg->max_iterations; ++k) {
        op(ctx, p, q);
        res->spmv_calls++;
        const double pq = dot(n, p, q);
        if (!isfinite(pq) || pq <= 0.0) {
            status = 2;
            goto done;
        }
        const double alpha = rz / pq;
        vc.alpha = alpha;
        vec_op(&vc, EW_XR, threads, n);
        if (cfg->recompute_interval > 0 && k % cfg->recompute_interval == 0) {
            op(ctx, x, q);
            res->spmv_calls++;
            vec_op(&vc, EW_RESID, threads, n);
        }
        if (!vec_finite(&vc, threads, n)) {
            status = 2;
            goto done;
        }
        res->iterations = k;
        const double rel = sqrt(dot(n, r, r)) / bnorm;
        history[h++] = rel;
        if (rel > cfg->divergence_limit) {
            status = 2;
            goto done;
        }
        if (rel <= cfg->rel_tolerance) {
            res->converged = 1;
            goto done;
        }
        vec_op(&vc, EW_PRECOND, threads, n);
        const double rz_new = dot(n, r, z);
        const double beta = rz_new / rz;
        vc.beta = beta;
        vec_op(&vc, EW_PUPD, threads, n);
        rz = rz_new;
    }
    res->converged = 0;
done:
    res->history_len = h;
    free(r);
    free(z);
    free(p);
    free(q);
    return status;
}

/* cg.cpp:121-132 */
int ewo_compute_alpha(double t_reorder, double t_kernel, double t_base, int64_t* alpha,
                      int* finite) {
    if (!(t_reorder >= 0.0 && t_kernel >= 0.0 && t_base >= 0.0)) return 1;
    *alpha = -1;
    *finite = 0;
    if (t_kernel >= t_base) return 0;
    const double ratio = t_reorder / (t_base - t_kernel);
    const int64_t a = (int64_t)ceil(ratio);
    *alpha = a > 1 ? a : 1;
    *finite = 1;
    return 0;
}

void ewo_csr_op(void* ctx, const double* x, double* y) {
    const ewo_csr_ctx* c = (const ewo_csr_ctx*)ctx;
    ewo_spmv_csr(c->nrows, c->ncols, c->ro, c->ci, c->v, x, y);
}

void ewo_layout_op(void* ctx, const double* x, double* y) {
    const ewo_layout_ctx* c = (const ewo_layout_ctx*)ctx;
    ewo_spmv_layout(c->l, x, c->scatter, y);
}

/* cg.cpp:106-119 cg_solve_permuted when permuted != 0: b and diag are
 * permuted once on entry (apply_forward), the solution once on exit
 * (apply_inverse). */
int ewo_cg_layout(const ewo_layout* l, int permuted, int64_t n, const double* b,
                  const double* diag, const ewo_cg_config* cfg, double* x, double* history,
                  ewo_cg_result* res) {
    return ewo_cg_layout_mt(l, permuted, n, b, diag, cfg, x, history, res, 1);
}

/* ewo_cg_layout with the layout SpMV split over warps and the element-wise
 * loops over rows on `threads` threads: each row's sum and each dot product
 * are the single-threaded ones, so results are bit-identical for any thread
 * count (the config-4 parity check runs 1000+ iterations of 5M rows). */
int ewo_cg_layout_mt(const ewo_layout* l, int permuted, int64_t n, const double* b,
                     const double* diag, const ewo_cg_config* cfg, double* x, double* history,
                     ewo_cg_result* res, int threads) {
    ewo_layout_mt_ctx ctx = {l, permuted ? 0 : 1, threads};
    if (!permuted)
        return ewo_cg_solve_mt(ewo_layout_op_mt, &ctx, n, b, diag, cfg, x, history, res, threads);
    double* bp = (double*)malloc(sizeof(double) * (size_t)(n + 1));
    double* dp = diag ? (double*)malloc(sizeof(double) * (size_t)(n + 1)) : NULL;
    double* xp = (double*)malloc(sizeof(double) * (size_t)(n + 1));
    for (int64_t k = 0; k < n; ++k) {
        bp[k] = b[l->forward[k]];
        if (dp) dp[k] = diag[l->forward[k]];
    }
    const int st = ewo_cg_solve_mt(ewo_layout_op_mt, &ctx, n, bp, dp, cfg, xp, history, res, threads);
    for (int64_t k = 0; k < n; ++k) x[l->forward[k]] = xp[k];
    free(bp);
    free(dp);
    free(xp);
    return st;
}

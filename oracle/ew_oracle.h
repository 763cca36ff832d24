/* CPU restatement of the reference's ELL-WARP hot path (arXiv 1501.00324),
 * in plain C99.
 *
 * TEST INFRASTRUCTURE ONLY: this is the checker for the B200 library, used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg. It is never
 * linked into or called from paper_1501_00324_b200/.
 *
 * Parity of this restatement is pinned two ways (tests/test_oracle.py):
 *   1. against the golden vectors the reference's own tests hold
 *      (proj/tests/test_ellwarp.cpp, test_solver.cpp, acceptance.cpp,
 *      python/tests/test_smoke.py), committed under tests/golden/;
 *   2. against the real reference compiled from its sources by
 *      oracle/Makefile into oracle/_ref/libellwarp_ref.so, on the reference's
 *      own randomized corpus (tests/test_support.hpp random_case).
 *
 * Types follow proj/include/ellwarp/types.hpp:13-14 (idx = int64, real = double).
 */
#ifndef EW_ORACLE_H
#define EW_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes: 0 ok, 1 invalid argument (std::invalid_argument),
 * 2 CG divergence (CgDivergenceError). */

/* row-parallel (pthreads) port of spmv_csr_reference (bench CPU comparison only) */
int ewo_spmv_csr_mt(int64_t nrows, int64_t ncols, const int64_t* ro, const int64_t* ci,
                    const double* v, const double* x, double* y, int threads);
/* csr.cpp:75-86 spmv_csr_reference */
int ewo_spmv_csr(int64_t nrows, int64_t ncols, const int64_t* ro, const int64_t* ci,
                 const double* v, const double* x, double* y);
/* csr.cpp:106-117 extract_diagonal */
void ewo_extract_diagonal(int64_t nrows, int64_t ncols, const int64_t* ro, const int64_t* ci,
                          const double* v, double* d);
/* csr.cpp:57-73 validate_csr: 0 valid, 1 invalid */
int ewo_validate_csr(int64_t nrows, int64_t ncols, int64_t nro, const int64_t* ro, int64_t nnz,
                     const int64_t* ci);
/* permutation.cpp:49-55 sort_rows_desc */
void ewo_sort_rows_desc(int64_t nrows, const int64_t* ro, int64_t* fwd, int64_t* inv);
/* warp_layout.cpp:76-84 compute_k2_lanes; returns -1 on invalid arguments */
int64_t ewo_compute_k2_lanes(int64_t nnz_row, int64_t threshold, int64_t warp_size);

/* WarpLayoutK1 / WarpLayoutK2 (warp_layout.hpp:13-61) in one struct; the
 * K2-only arrays are NULL for K1. */
typedef struct {
    int kind; /* 1 = K1, 2 = K2 */
    int64_t warp_size, nrows, ncols, nnz, threshold, nwarps, nslots;
    int row_major;
    double* values;
    int64_t* col_indices;
    int64_t* warp_offset;
    int64_t* maxrows;
    int64_t* rows_in_warp;
    int64_t* reduction;        /* K2 */
    int64_t* rows_offset_warp; /* K2 */
    int64_t* forward;          /* row_perm.forward */
    int64_t* inverse;
    int64_t* sorted_row_length;
} ewo_layout;

/* warp_layout.cpp:32-74 build_k1 / :86-147 build_k2. Returns 0 or 1. */
int ewo_build_k1(int64_t nrows, int64_t ncols, const int64_t* ro, const int64_t* ci,
                 const double* v, int warp_size, int segment_bytes, int align, int sort_rows,
                 int row_major, ewo_layout** out);
int ewo_build_k2(int64_t nrows, int64_t ncols, const int64_t* ro, const int64_t* ci,
                 const double* v, int warp_size, int segment_bytes, int align, int64_t threshold,
                 int sort_rows, ewo_layout** out);
void ewo_layout_free(ewo_layout* l);
int64_t ewo_layout_stored_slots(const ewo_layout* l);
/* warp_layout.cpp:149-174 value_slot_map */
void ewo_value_slot_map(const ewo_layout* l, const int64_t* ro, int64_t* map);

/* warp_spmv.cpp:9-60 run_k1 and :62-126 run_k2; scatter = 1 stores through
 * row_perm.forward (K1/K2), 0 stores in sorted numbering (the *_sorted kernels). */
void ewo_spmv_layout(const ewo_layout* l, const double* x, int scatter, double* y);

/* reorder.cpp:8-43 make_reordered_r (+ make_reordered_rs when sort_within_rows).
 * Output arrays have the input's shapes. Returns 1 for non-square input. */
int ewo_reorder(int64_t nrows, int64_t ncols, const int64_t* ro, const int64_t* ci,
                const double* v, const int64_t* fwd, const int64_t* inv, int sort_within_rows,
                int64_t* ci_out, double* v_out);

/* cg.cpp:25-104 cg_solve against an operator callback. */
typedef void (*ewo_spmv_fn)(void* ctx, const double* x, double* y);
typedef struct {
    double rel_tolerance;
    int64_t max_iterations;
    int jacobi;
    int64_t recompute_interval;
    double divergence_limit;
} ewo_cg_config;
typedef struct {
    int64_t iterations;
    int converged;
    int64_t spmv_calls;
    int64_t history_len;
} ewo_cg_result;
/* history must hold max_iterations + 1 entries. */
int ewo_cg_solve(ewo_spmv_fn op, void* ctx, int64_t n, const double* b, const double* diag,
                 const ewo_cg_config* cfg, double* x, double* history, ewo_cg_result* res);

/* cg.cpp:121-132 compute_alpha; *finite = 0 means infinity. */
int ewo_compute_alpha(double t_reorder, double t_kernel, double t_base, int64_t* alpha,
                      int* finite);

/* Convenience operators for ewo_cg_solve. */
typedef struct {
    int64_t nrows, ncols;
    const int64_t *ro, *ci;
    const double* v;
} ewo_csr_ctx;
void ewo_csr_op(void* ctx, const double* x, double* y);
typedef struct {
    const ewo_layout* l;
    int scatter;
} ewo_layout_ctx;
void ewo_layout_op(void* ctx, const double* x, double* y);
/* Multi-threaded forms for full-size parity runs: warps (SpMV) and rows
 * (CG vector updates) split over threads, dot products sequential; bitwise
 * equal to the single-threaded functions for any thread count. */
typedef struct {
    const ewo_layout* l;
    int scatter;
    int threads;
} ewo_layout_mt_ctx;
void ewo_layout_op_mt(void* ctx, const double* x, double* y);
void ewo_spmv_layout_mt(const ewo_layout* l, const double* x, int scatter, double* y, int threads);
int ewo_cg_solve_mt(ewo_spmv_fn op, void* ctx, int64_t n, const double* b, const double* diag,
                    const ewo_cg_config* cfg, double* x, double* history, ewo_cg_result* res,
                    int threads);

/* One CG over csr / layout operators chosen by id, as the reference's
 * _ellwarp.cg_solve binding does (module.cpp:227-249); permuted selects
 * cg_solve_permuted (cg.cpp:106-119) for layouts built on the r/rs operand. */
int ewo_cg_layout(const ewo_layout* l, int permuted, int64_t n, const double* b,
                  const double* diag, const ewo_cg_config* cfg, double* x, double* history,
                  ewo_cg_result* res);
int ewo_cg_layout_mt(const ewo_layout* l, int permuted, int64_t n, const double* b,
                     const double* diag, const ewo_cg_config* cfg, double* x, double* history,
                     ewo_cg_result* res, int threads);

#ifdef __cplusplus
}
#endif
#endif

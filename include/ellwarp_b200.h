/*
 * ellwarp_b200.h -- C ABI of the B200-native ELL-WARP SpMV + Jacobi-PCG library
 * (arXiv 1501.00324, Wong/Kuhl/Darve). Plain pointers and sizes only; no C++
 * or torch types cross this boundary.
 *
 * Every entry point replaces one call of the reference C++ library
 * (/root/reference/proj, cited as file:line below). The reference is a
 * single-threaded CPU emulation of the paper's GPU kernels; this library runs
 * the same algorithms as sm_100a CUDA kernels on device-resident data.
 *
 * Conventions
 *  - Status codes map 1:1 onto the reference's exceptions:
 *      EW_INVALID_ARGUMENT  <-> std::invalid_argument      (types.hpp:16-18)
 *      EW_CG_DIVERGENCE     <-> ellwarp::CgDivergenceError (cg.hpp:28-30)
 *    EW_UNSUPPORTED marks inputs the device path rejects (a WarpTracer, ids of
 *    the baseline formats, > 2^31-1 rows/columns), EW_CUDA a CUDA failure.
 *    ew_last_error() returns the message of the calling thread's last error.
 *  - Index types at the boundary are the reference's (int64 idx, double
 *    real; types.hpp:13-14). On the device columns and permutations are
 *    int32 and slot offsets int64 ("Data layout in HBM").
 *  - mem_kind says where x / y / b / solution buffers live. EW_MEM_HOST
 *    buffers are copied on `stream` and the call returns after the result
 *    is back on the host (the reference returns a fresh std::vector).
 *    EW_MEM_DEVICE buffers are device pointers; the call is asynchronous on
 *    `stream` (a cudaStream_t; NULL = legacy default stream).
 *  - Handles are immutable after creation except through the explicit
 *    *_refresh_values calls; distinct handles may be used concurrently from
 *    different threads, as the reference's kernels are pure.
 */
#ifndef ELLWARP_B200_H
#define ELLWARP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EW_ABI_VERSION 1

typedef enum ew_status {
    EW_OK = 0,
    EW_INVALID_ARGUMENT = 1,
    EW_CG_DIVERGENCE = 2,
    EW_UNSUPPORTED = 3,
    EW_CUDA = 4,
    EW_OUT_OF_MEMORY = 5
} ew_status;

typedef enum ew_mem_kind { EW_MEM_HOST = 0, EW_MEM_DEVICE = 1 } ew_mem_kind;

typedef enum ew_layout_kind { EW_LAYOUT_K1 = 1, EW_LAYOUT_K2 = 2 } ew_layout_kind;

typedef struct ew_csr_t* ew_csr;       /* device-resident SparseCsr (csr.hpp:26-36)   */
typedef struct ew_layout_t* ew_layout; /* device WarpLayoutK1/K2 (warp_layout.hpp:13-61) */
typedef struct ew_kernel_t* ew_kernel; /* PreparedKernel (kernels.hpp:16-23)          */

/* WarpModelConfig (warp_model.hpp:16-25). block_size, ideal_cache and
 * cache_lines are validated like the reference but do not change results. */
typedef struct ew_warp_config {
    int32_t warp_size;          /* power of two; default 32 */
    int32_t block_size;         /* multiple of warp_size; default 128 */
    int32_t segment_bytes;      /* power of two; default 128 */
    int32_t align_warp_offsets; /* default 1 */
    int32_t ideal_cache;        /* default 0 */
    int32_t cache_lines;        /* > 0; default 64 */
} ew_warp_config;

/* KernelOptions (kernels.hpp:29-32) */
typedef struct ew_kernel_options {
    int64_t k2_threshold; /* <= 0: max row length (kernels.cpp:16-21) */
    int64_t hyb_k_ell;    /* < 0: 2/3 coverage heuristic */
    /* Row order of the r / rs kernels (extension; the reference has only
     * EW_ROW_ORDER_REFERENCE). EW_ROW_ORDER_LOCALITY: the stable longest-first
     * sort is applied to a Cuthill-McKee order instead of the row ids, so
     * mesh neighbours share a warp; every row keeps the reference's entry
     * order (same row sums), the permutation -- and apply_permuted's
     * numbering -- is that order. */
    int64_t row_order;
} ew_kernel_options;

enum { EW_ROW_ORDER_REFERENCE = 0, EW_ROW_ORDER_LOCALITY = 1 };

/* CgConfig (cg.hpp:10-18) */
typedef struct ew_cg_config {
    double rel_tolerance;       /* default 1e-8 */
    int64_t max_iterations;     /* default 1000 */
    int32_t jacobi;             /* default 1 */
    int64_t recompute_interval; /* default 50 */
    double divergence_limit;    /* default 1e6 */
} ew_cg_config;

/* CgResult (cg.hpp:20-26); history is returned through a caller buffer of
 * max_iterations + 1 doubles. */
typedef struct ew_cg_result {
    int64_t iterations;
    int32_t converged;
    int64_t spmv_calls;
    int64_t history_len;
} ew_cg_result;

typedef struct ew_layout_info {
    int32_t kind; /* ew_layout_kind */
    int32_t warp_size;
    int32_t row_major;
    int32_t sorted;
    int64_t nrows, ncols, nnz;
    int64_t nwarps;
    int64_t nslots;       /* flat array length, incl. alignment gaps */
    int64_t stored_slots; /* WarpLayoutK1/K2::stored_slots (warp_layout.cpp:20-29) */
    int64_t threshold;    /* K2 only */
    int64_t device_bytes; /* HBM held by the layout */
    int64_t narrow_slots; /* K1: slots whose columns stream as 16-bit offsets
                             from a per-warp base (0: all int32) */
    int64_t col_stream_bytes; /* column bytes one SpMV launch streams (int32,
                                 16-bit, or shared per lane group) */
} ew_layout_info;

/* Host views of a layout, in the reference's int64/double element types.
 * Any pointer may be NULL (skipped). Sizes: values/col_indices nslots;
 * per-warp arrays nwarps; forward/sorted_row_length nrows. */
typedef struct ew_layout_arrays {
    double* values;
    int64_t* col_indices;
    int64_t* warp_offset;
    int64_t* maxrows;
    int64_t* rows_in_warp;
    int64_t* reduction;        /* K2 */
    int64_t* rows_offset_warp; /* K2 */
    int64_t* forward;          /* row_perm.forward */
    int64_t* inverse;          /* row_perm.inverse */
    int64_t* sorted_row_length;
} ew_layout_arrays;

/* Host description used to import an externally built layout, so
 * spmv_k1(const WarpLayoutK1&, x) (warp_spmv.hpp:11-23) can run on the device
 * for any layout the C++ API hands it. Arrays as in ew_layout_arrays. */
typedef struct ew_layout_desc {
    int32_t kind;
    int32_t warp_size;
    int32_t row_major;
    int64_t nrows, ncols, nnz, nwarps, nslots, threshold;
    const double* values;
    const int64_t* col_indices;
    const int64_t* warp_offset;
    const int64_t* maxrows;
    const int64_t* rows_in_warp;
    const int64_t* reduction;        /* K2; NULL for K1 */
    const int64_t* rows_offset_warp; /* K2; NULL for K1 */
    const int64_t* forward;
    const int64_t* sorted_row_length;
} ew_layout_desc;

typedef struct ew_kernel_info {
    char id[16];
    int64_t nrows, ncols, nnz;
    int64_t stored_slots; /* PreparedKernel::stored_slots (kernels.hpp:22) */
    int64_t nwarps;       /* 0 for csr_ref */
    int32_t has_perm;     /* PreparedKernel::perm set (r/rs variants) */
    int32_t layout_kind;  /* 0 = csr_ref, else ew_layout_kind */
    int64_t device_bytes;
    int64_t narrow_slots; /* as ew_layout_info::narrow_slots */
    int64_t col_stream_bytes; /* as ew_layout_info::col_stream_bytes */
} ew_kernel_info;

/* ---- errors / library ---------------------------------------------------- */
const char* ew_last_error(void);
const char* ew_status_string(ew_status s);
int32_t ew_abi_version(void);
/* kernel_ids() (kernels.cpp:7-12): 11 ids in the reference's order. */
int32_t ew_kernel_id_count(void);
const char* ew_kernel_id(int32_t i);
/* 1 if the id runs on the device in this build, 0 if it is a known id the
 * device path does not implement yet (EW_UNSUPPORTED), -1 if unknown. */
int32_t ew_kernel_id_supported(const char* id);
/* Count of this library's kernel launches since load (all streams). */
int64_t ew_launch_count(void);
/* Benchmark helper, stream-ordered L2 flush: reads `bytes` of the device
 * buffer `buf` (pass >= 2x the L2 size) with an L2 evict_last policy, so it
 * also displaces the lines the SpMV kernels tag evict_last (the x gathers),
 * which a plain read of a large buffer would not. */
ew_status ew_l2_flush(const void* buf, int64_t bytes, void* stream);

/* ---- matrices (csr.hpp / csr.cpp) --------------------------------------- */
/* Upload + validate_csr (csr.cpp:57-73) on the device. Row offsets and
 * column ranges are always checked (memory safety); the strictly-increasing
 * column check runs with EW_CSR_CANONICAL. Without it the matrix may hold a
 * renumbered r operand (reorder.hpp:17), which the reference feeds to
 * build_k1 / build_k2 unsorted. */
#define EW_CSR_CANONICAL 1
ew_status ew_csr_create(int64_t nrows, int64_t ncols, int64_t n_row_offsets,
                        const int64_t* row_offsets, int64_t nnz, const int64_t* col_indices,
                        const double* values, ew_mem_kind mem, int32_t flags, void* stream,
                        ew_csr* out);
ew_status ew_csr_destroy(ew_csr m);
ew_status ew_csr_shape(ew_csr m, int64_t* nrows, int64_t* ncols, int64_t* nnz);
ew_status ew_csr_export(ew_csr m, int64_t* row_offsets, int64_t* col_indices, double* values);
/* Replace the values (same structure); the values-only refresh input. */
ew_status ew_csr_update_values(ew_csr m, const double* values, ew_mem_kind mem, void* stream);
/* spmv_csr_reference (csr.cpp:75-86) on the device, bit-identical. */
ew_status ew_csr_spmv(ew_csr m, const double* x, int64_t nx, double* y, int64_t ny,
                      ew_mem_kind mem, void* stream);
/* extract_diagonal (csr.cpp:106-117). */
ew_status ew_csr_extract_diagonal(ew_csr m, double* diag, ew_mem_kind mem, void* stream);

/* ---- permutation / reorder (permutation.hpp, reorder.hpp) ---------------- */
/* sort_rows_desc (permutation.cpp:49-55): stable, longest first. Host out. */
ew_status ew_sort_rows_desc(ew_csr m, int64_t* forward, int64_t* inverse);
/* make_reordered_r (reorder.cpp:8-17), + make_reordered_rs (:19-43) when
 * sort_within_rows. forward_in (host, nrows) is the permutation to renumber
 * by (Permutation::from_forward checks, permutation.cpp:17-28); NULL means
 * sort_rows_desc(m), as prepare_kernel does (kernels.cpp:26). forward_out
 * (host, nrows, nullable) receives the permutation used. */
ew_status ew_reorder(ew_csr m, const int64_t* forward_in, int32_t sort_within_rows, ew_csr* out,
                     int64_t* forward_out);
/* The per-row (column, value) sort of make_reordered_rs on its own
 * (reorder.cpp:26-41): columns ascending within every row. */
ew_status ew_csr_sort_rows(ew_csr m, ew_csr* out);
/* apply_forward (permutation.cpp:35-40): out[k] = in[forward[k]], or with
 * inverse = 1 apply_inverse (:42-47): out[forward[k]] = in[k].
 * forward is host int64[n]; in/out live in `mem`. */
ew_status ew_permute(const int64_t* forward, int64_t n, const double* in, double* out,
                     int32_t inverse, ew_mem_kind mem, void* stream);
/* compute_k2_lanes (warp_layout.cpp:76-84) */
ew_status ew_compute_k2_lanes(int64_t nnz_row, int64_t threshold, int64_t warp_size,
                              int64_t* lanes);

/* ---- layouts (warp_layout.hpp) ------------------------------------------ */
/* build_k1 (warp_layout.cpp:32-74) / build_k2 (:86-147), built on the device.
 * threshold is used for K2 only; row_major for K1 only (BuildOptions). */
ew_status ew_layout_build(ew_csr m, int32_t kind, const ew_warp_config* cfg, int64_t threshold,
                          int32_t sort_rows, int32_t row_major, ew_layout* out);
ew_status ew_layout_import(const ew_layout_desc* desc, ew_layout* out);
ew_status ew_layout_destroy(ew_layout l);
ew_status ew_layout_get_info(ew_layout l, ew_layout_info* info);
ew_status ew_layout_export(ew_layout l, const ew_layout_arrays* out);
/* value_slot_map (warp_layout.cpp:149-174); map is host int64[nnz]. */
ew_status ew_layout_value_slot_map(ew_layout l, ew_csr m, int64_t* map);
/* Values-only refresh through the slot map (the paper's per-Newton-iteration
 * reorder): the layout's values are rewritten from m's
 * current values; m must have the structure the layout was built from. */
ew_status ew_layout_refresh_values(ew_layout l, ew_csr m, void* stream);
/* dump_layout (warp_layout.cpp:185-207); *len gets strlen + 1. */
ew_status ew_layout_dump(ew_layout l, char* buf, size_t cap, size_t* len);
/* spmv_k1 / spmv_k1_sorted / spmv_k2 / spmv_k2_sorted (warp_spmv.cpp:130-146):
 * scatter = 1 stores y in original numbering through row_perm.forward. */
ew_status ew_layout_spmv(ew_layout l, const double* x, int64_t nx, double* y, int64_t ny,
                         int32_t scatter, ew_mem_kind mem, void* stream);

/* ---- prepared kernels (kernels.hpp) -------------------------------------- */
/* prepare_kernel (kernels.cpp:59-125). opts may be NULL (defaults). */
ew_status ew_kernel_prepare(const char* id, ew_csr m, const ew_warp_config* cfg,
                            const ew_kernel_options* opts, ew_kernel* out);
ew_status ew_kernel_destroy(ew_kernel k);
ew_status ew_kernel_get_info(ew_kernel k, ew_kernel_info* info);
/* PreparedKernel::perm (r/rs only); host int64[nrows] each, nullable. */
ew_status ew_kernel_get_perm(ew_kernel k, int64_t* forward, int64_t* inverse);
/* The kernel's layout (NULL for csr_ref); owned by the kernel. */
ew_status ew_kernel_get_layout(ew_kernel k, ew_layout* out);
/* PreparedKernel::apply: y = A x in original numbering. */
ew_status ew_kernel_apply(ew_kernel k, const double* x, int64_t nx, double* y, int64_t ny,
                          ew_mem_kind mem, void* stream);
/* PreparedKernel::apply_permuted (r/rs only): x, y in sorted numbering. */
ew_status ew_kernel_apply_permuted(ew_kernel k, const double* x, int64_t nx, double* y,
                                   int64_t ny, ew_mem_kind mem, void* stream);
/* Values-only refresh of a prepared kernel from m (same structure). */
ew_status ew_kernel_refresh_values(ew_kernel k, ew_csr m, void* stream);

/* ---- Jacobi PCG (cg.hpp / cg.cpp) ---------------------------------------- */
/* cg_solve (cg.cpp:25-104) with the kernel's apply as operator, entirely on
 * the device. diag may be NULL when cfg->jacobi == 0 (else it is required,
 * as in the reference). history: host double[max_iterations + 1].
 * Solution x is written in `mem`. */
ew_status ew_cg_solve(ew_kernel k, const double* b, const double* diag, int64_t n,
                      const ew_cg_config* cfg, ew_mem_kind mem, double* x, double* history,
                      ew_cg_result* result, void* stream);
/* cg_solve_permuted (cg.cpp:106-119) with the kernel's apply_permuted (r/rs
 * kernels): b, diag and the solution are in original numbering. */
ew_status ew_cg_solve_permuted(ew_kernel k, const double* b, const double* diag, int64_t n,
                               const ew_cg_config* cfg, ew_mem_kind mem, double* x,
                               double* history, ew_cg_result* result, void* stream);
/* cg_solve (cg.cpp:25-104) with an arbitrary operator, the reference's
 * SpmvFn closure (cg.hpp:32). The callback gets x (input) and y (output),
 * both of length n, in op_mem (EW_MEM_HOST: the solver stages them through
 * host buffers, so a std::function over std::span works unchanged;
 * EW_MEM_DEVICE: device pointers, work may be enqueued on `stream`). It
 * returns 0 on success or an ew_status. The solver's vector work and dots
 * stay on the device; it synchronises before each callback. */
typedef int (*ew_operator_fn)(void* ctx, const double* x, double* y, void* stream);
ew_status ew_cg_solve_operator(ew_operator_fn op, void* ctx, ew_mem_kind op_mem, const double* b,
                               const double* diag, int64_t n, const ew_cg_config* cfg,
                               ew_mem_kind mem, double* x, double* history, ew_cg_result* result,
                               void* stream);
/* ---- row-partitioned operator and CG (no reference
 * counterpart: the reference is single-threaded) -------------------------
 * Partition: contiguous nnz-balanced row blocks, bounds[g] = first row whose
 * nnz prefix reaches g * nnz / nparts (bounds has nparts + 1 entries). */
ew_status ew_partition_rows(const int64_t* row_offsets, int64_t nrows, int32_t nparts, int64_t* bounds);
/* 128-byte ncclUniqueId for ew_dist_create (broadcast it to every rank). */
ew_status ew_nccl_unique_id(void* id);
typedef struct ew_dist_t* ew_dist;
/* Partitions [first_part, first_part + local_parts) of the square global
 * host CSR, each with a local operator `kernel_id` (k1, k2, csr_ref or a
 * baseline; r/rs ids need a square local matrix and are rejected).
 * nccl_id != NULL: NCCL transport, one partition per process
 * (local_parts = 1, first_part = rank, nparts = world size).
 * nccl_id == NULL: every partition in this process on the current device
 * (first_part = 0, local_parts = nparts), halos as device copies.
 * bounds may be NULL (ew_partition_rows). */
ew_status ew_dist_create(int64_t nrows, int64_t ncols, int64_t n_row_offsets, const int64_t* row_offsets,
                         int64_t nnz, const int64_t* col_indices, const double* values,
                         const int64_t* bounds, int32_t nparts, int32_t first_part,
                         int32_t local_parts, const void* nccl_id, const char* kernel_id,
                         const ew_warp_config* cfg, const ew_kernel_options* opts, void* stream,
                         ew_dist* out);
/* Scalable constructor (NCCL only): this rank passes just its own row block
 * [bounds[rank], bounds[rank+1]) of the global matrix, with GLOBAL column
 * ids (row_offsets starts at 0, nrows_local + 1 entries). Ghost requests are
 * exchanged over NCCL at setup. */
ew_status ew_dist_create_block(int64_t nrows_global, int64_t nrows_local, const int64_t* row_offsets,
                               const int64_t* col_indices, const double* values,
                               const int64_t* bounds, int32_t nparts, int32_t rank,
                               const void* nccl_id, const char* kernel_id,
                               const ew_warp_config* cfg, const ew_kernel_options* opts,
                               void* stream, ew_dist* out);
/* Peer transport, every partition in this process on the current device:
 * the same push / mailbox kernels as the IPC transport, peers being the
 * process's own partitions (tests the NVLink protocol on one GPU). */
ew_status ew_dist_create_peer(int64_t nrows, int64_t ncols, int64_t n_row_offsets, const int64_t* row_offsets,
                              int64_t nnz, const int64_t* col_indices, const double* values,
                              const int64_t* bounds, int32_t nparts, const char* kernel_id,
                              const ew_warp_config* cfg, const ew_kernel_options* opts, void* stream,
                              ew_dist* out);
/* Rank-ordered allgather supplied by the caller (e.g. torch.distributed):
 * recv receives world_size * bytes, rank g's send at offset g * bytes.
 * Returns 0 on success. */
typedef int (*ew_allgather_fn)(const void* send, void* recv, size_t bytes, void* user);
/* One partition per process, peers reached through CUDA IPC mappings of each
 * other's ghost buffers and mailboxes (NVLink stores; no NCCL on the data
 * path). Same arguments as ew_dist_create_block, with the allgather used for
 * setup (ghost requests, IPC handles). Collective: every rank calls it, and
 * every rank destroys its operator only after the last solve on all ranks. */
ew_status ew_dist_create_block_ipc(int64_t nrows_global, int64_t nrows_local, const int64_t* row_offsets,
                                   const int64_t* col_indices, const double* values, const int64_t* bounds,
                                   int32_t nparts, int32_t rank, ew_allgather_fn allgather, void* user,
                                   const char* kernel_id, const ew_warp_config* cfg,
                                   const ew_kernel_options* opts, void* stream, ew_dist* out);
/* The setup exchange of ew_dist_create_block_ipc for this rank's row block,
 * on the host only (no device work; a collective through the allgather):
 * the block's ghost columns (ascending, hence grouped by owner) and, per peer
 * h, the global rows of this block h needs, send_rows[send_off[h],
 * send_off[h+1]). ghosts: capacity >= row_offsets[nrows_local]; send_off:
 * nparts + 1; send_rows: capacity >= nrows_local * nparts. */
ew_status ew_dist_plan_block(int64_t nrows_local, const int64_t* row_offsets, const int64_t* col_indices,
                             const int64_t* bounds, int32_t nparts, int32_t rank, ew_allgather_fn allgather,
                             void* user, int64_t* nghost, int64_t* ghosts, int64_t* send_off, int64_t* send_rows);
ew_status ew_dist_destroy(ew_dist d);
/* Row range, ghost count and send count of local partition i. */
ew_status ew_dist_get_info(ew_dist d, int32_t local_index, int64_t* row_begin, int64_t* row_end,
                           int64_t* nghost, int64_t* nsend);
/* Matrix bytes of local partition i's layouts (interior + boundary, or the
 * one local layout): stored slots, and the value + column bytes one SpMV
 * streams (8 per slot + 4 / 2 / grouped column bytes; csr_ref: 12 nnz). */
ew_status ew_dist_get_layout_bytes(ew_dist d, int32_t local_index, int64_t* stored_slots,
                                   int64_t* stream_bytes);
/* y = A x on this process's owned rows (concatenated in partition order). */
ew_status ew_dist_spmv(ew_dist d, const double* x, double* y, ew_mem_kind mem, void* stream);
/* cg_solve (cg.cpp:25-104) over the partitioned operator: halo exchange per
 * SpMV, all-gathered dot products summed in rank order. b, diag, x: owned
 * rows; history on every rank. */
ew_status ew_dist_cg_solve(ew_dist d, const double* b, const double* diag, const ew_cg_config* cfg,
                           ew_mem_kind mem, double* x, double* history, ew_cg_result* result,
                           void* stream);
/* ---- one process, several GPUs (SURVEY.md §8(b) ew_mgpu_cg_solve) ---------
 * The square host CSR (validate_csr ranges) split into ngpus nnz-balanced
 * row blocks (ew_partition_rows); block g lives on device devices[g]
 * (NULL: device g; a device may repeat, e.g. every block on device 0 for
 * tests: then set CUDA_DEVICE_MAX_CONNECTIONS >= 2 per block on the device
 * before the first CUDA call, the blocks' streams wait on each other and
 * need a hardware queue each). Peers are reached by peer access (NVLink stores) with the same
 * push / mailbox / rank-ordered reduction kernels as the CUDA-IPC
 * transport, one host thread and stream per block. Replaces running
 * ew_dist_create_block_ipc on ngpus processes for callers that are one
 * process (the reference's CLI `cg`, tools/ellwarp_cli.cpp:186-213; FEM time
 * stepping, fem/timestep.cpp:90-107). */
typedef struct ew_mgpu_t* ew_mgpu;
ew_status ew_mgpu_create(int64_t nrows, const int64_t* row_offsets, const int64_t* col_indices, const double* values,
                         int32_t ngpus, const int32_t* devices, const char* kernel_id, const ew_warp_config* cfg,
                         const ew_kernel_options* opts, ew_mgpu* out);
ew_status ew_mgpu_destroy(ew_mgpu m);
/* y = A x; x, y host arrays of nrows. */
ew_status ew_mgpu_spmv(ew_mgpu m, const double* x, double* y);
/* cg_solve (cg.cpp:25-104) over the blocks; b, diag, x host arrays of nrows,
 * history max_iterations + 1 entries (may be NULL). */
ew_status ew_mgpu_cg_solve(ew_mgpu m, const double* b, const double* diag, const ew_cg_config* cfg, double* x,
                           double* history, ew_cg_result* result);
/* ---- FEM assembly as K1 row sums (fem/assembly.cpp:38-159, SURVEY.md
 * §8(f) #3) ---------------------------------------------------------------
 * build_assembly_map on the device: the node-adjacency pattern of the
 * tetrahedra (elements: int64[nelements * 4], host), one contribution row per
 * pattern entry / per node in element-major order, packed into K1 layouts. */
typedef struct ew_assembly_t* ew_assembly;
ew_status ew_assembly_create(int64_t nelements, const int64_t* elements, int64_t nnodes,
                             const ew_warp_config* cfg, ew_assembly* out);
ew_status ew_assembly_destroy(ew_assembly a);
/* The tangent pattern (host; arrays nullable, call with NULL to size). */
ew_status ew_assembly_pattern(ew_assembly a, int64_t* nnz, int64_t* row_offsets,
                              int64_t* col_indices);
/* assemble_spmv (fem/assembly.cpp:140-159): ke = element tangents
 * [nelements][4][4], re = element residuals [nelements][4]; outputs the
 * tangent values in pattern order and the residual (either may be NULL).
 * Bit-identical to the reference's scatter + row sum. */
ew_status ew_assembly_run(ew_assembly a, const double* ke, const double* re,
                          double* tangent_values, double* residual, ew_mem_kind mem,
                          void* stream);
/* The same, but the tangent lands directly in the slots of kernel k (an
 * ELL-WARP kernel prepared on the pattern): no values refresh before the
 * next SpMV / CG. */
ew_status ew_assembly_run_into(ew_assembly a, const double* ke, const double* re, ew_kernel k,
                               double* residual, ew_mem_kind mem, void* stream);
/* compute_alpha (cg.cpp:121-132); *finite = 0 means infinity. */
ew_status ew_compute_alpha(double t_reorder, double t_kernel, double t_base, int64_t* alpha,
                           int32_t* finite);

#ifdef __cplusplus
}
#endif
#endif /* ELLWARP_B200_H */

// Internal types shared by the CUDA translation units of libellwarp_b200.so.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "ellwarp_b200.h"

namespace ew {

// Raised inside the library, converted to an ew_status at the C boundary.
struct Error : std::runtime_error {
    ew_status status;
    Error(ew_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

inline void require(bool cond, const std::string& msg) {
    if (!cond) throw Error(EW_INVALID_ARGUMENT, msg);
}

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        const ew_status s = (e == cudaErrorMemoryAllocation) ? EW_OUT_OF_MEMORY : EW_CUDA;
        throw Error(s, std::string(what) + ": " + cudaGetErrorString(e));
    }
}
#define EW_CUDA_CHECK(expr) ::ew::cuda_check((expr), #expr)

// Launch accounting (the bench's gpu_launches claim and the smoke checks).
extern std::atomic<int64_t> g_launches;
inline void launched(const char* what) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    cuda_check(cudaGetLastError(), what);
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Programmatic dependent launch: a kernel launched with launch_pdl may be
// scheduled while the previous kernel on the stream drains; it must call
// pdl_wait() before touching anything that kernel wrote. Kernels on the CG
// path call pdl_trigger() on entry so their successor can launch early. Both
// are no-ops for kernels launched without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

bool pdl_enabled();  // EW_PDL=0 disables the attribute (A/B runs)

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), unsigned grid, unsigned block, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cuda_check(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...), "cudaLaunchKernelEx");
}

// Owning device allocation (cudaMalloc; long-lived data: matrices, layouts).
template <typename T>
class DevBuf {
  public:
    DevBuf() = default;
    explicit DevBuf(size_t n) { alloc(n); }
    ~DevBuf() { release(); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr, o.n_ = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p_ = o.p_, n_ = o.n_;
            o.p_ = nullptr, o.n_ = 0;
        }
        return *this;
    }
    // Contents are undefined after alloc (as cudaMalloc's); an allocation of
    // the same size is kept: cudaMalloc / cudaFree synchronise the device.
    void alloc(size_t n) {
        if (p_ && n == n_) return;
        release();
        n_ = n;
        if (n) EW_CUDA_CHECK(cudaMalloc(&p_, n * sizeof(T)));
    }
    void release() {
        if (p_) cudaFree(p_);
        p_ = nullptr;
        n_ = 0;
    }
    T* get() const { return p_; }
    size_t size() const { return n_; }
    size_t bytes() const { return n_ * sizeof(T); }

  private:
    T* p_ = nullptr;
    size_t n_ = 0;
};

// Keeps freed scratch (up to 8 GB) in the current device's default memory
// pool instead of returning it to the driver at every synchronisation (the
// default release threshold is 0: each call would re-map its scratch,
// ~0.1 ms).
void retain_pool();

// Loads every kernel of this library into the current device's context now.
// Under CUDA's default lazy loading a kernel's first launch loads it, and a
// load can wait for the device: a partition loading its SpMV or push kernel
// while a peer's kernel spins waiting for it deadlocks (seen with two
// partitions on one GPU). Every partitioned operator calls this before its
// first exchange. Once per device.
void load_all_kernels();
const void* kernel_anchor_assembly();
const void* kernel_anchor_dist();
const void* kernel_anchor_formats();
const void* kernel_anchor_kernel();
const void* kernel_anchor_layout();
const void* kernel_anchor_order();
const void* kernel_anchor_spmv();
const void* kernel_anchor_csr();

// Stream-ordered scratch (cudaMallocAsync from the device's default pool).
template <typename T>
class Scratch {
  public:
    Scratch(size_t n, cudaStream_t s) : s_(s), n_(n) {
        if (n) {
            retain_pool();
            EW_CUDA_CHECK(cudaMallocAsync(&p_, n * sizeof(T), s));
        }
    }
    ~Scratch() {
        if (p_) cudaFreeAsync(p_, s_);
    }
    Scratch(const Scratch&) = delete;
    Scratch& operator=(const Scratch&) = delete;
    T* get() const { return p_; }
    size_t size() const { return n_; }

  private:
    T* p_ = nullptr;
    cudaStream_t s_;
    size_t n_;
};

// Device-resident CSR: int64 row offsets, int32 columns, fp64 values.
struct CsrData {
    int64_t nrows = 0, ncols = 0, nnz = 0;
    int32_t maxrow = 0;
    DevBuf<int64_t> ro;
    DevBuf<int32_t> ci;
    DevBuf<double> v;
    size_t device_bytes() const { return ro.bytes() + ci.bytes() + v.bytes(); }
};

// Device ELL-WARP layout (K1 or K2). Per-warp metadata is int32 except the
// int64 slot offsets; columns and permutations are int32.
// Row-length bound of the cooperative head of a sorted K1 layout whose
// longest row exceeds 4x it (EW_K1_HEAD; 0 turns the split off).
int32_t head_mx();
struct LayoutData;
// The int32 column of every slot (nslots entries, alignment gaps 0) into
// out, from whatever form the layout holds (ew_layout.cu).
void decode_columns(const LayoutData& l, int32_t* out, cudaStream_t s);
// Gives a shrunk layout its full int32 slab back (the split-x boundary K1 of
// a partition reads it).
void restore_columns(LayoutData& l, cudaStream_t s);
// Whether layout_spmv / layout_spmv_dot read the full int32 slab for this
// layout (ew_spmv.cu).
bool spmv_reads_int32(const LayoutData& l);
void k1_long_setup();  // ew_spmv.cu: k1_long_kernel's shared-memory opt-in (current device)

// A second stream and fork / join events on the current device (RAII).
struct SideStream {
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    std::mutex mu;  // one fork ... join sequence at a time (callers on several host threads)
    SideStream() {
        EW_CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        EW_CUDA_CHECK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
        EW_CUDA_CHECK(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
    }
    ~SideStream() {
        if (join) cudaEventDestroy(join);
        if (fork) cudaEventDestroy(fork);
        if (s) cudaStreamDestroy(s);
    }
    SideStream(const SideStream&) = delete;
    SideStream& operator=(const SideStream&) = delete;
};

struct LayoutData {
    int kind = EW_LAYOUT_K1;
    int ws = 32;
    int ws_log2 = 5;
    int row_major = 0;
    int sorted = 1;  // rows sorted longest-first: active rows are a prefix
    int segment_bytes = 128;
    int align = 1;
    int64_t nrows = 0, ncols = 0, nnz = 0, nwarps = 0, nslots = 0, threshold = 0;
    int64_t n_active = 0;  // rows with at least one entry
    int64_t stored_slots = 0;
    int32_t max_reduction = 1;
    int32_t max_mx = 0;    // sorted K1: the longest warp's maxrows (0: unknown)
    // Sorted K1 with a few very long rows (power-law matrices): the leading
    // `head_warps` warps (rows over kHeadMx entries) run the cooperative K1
    // on `side` while the plain K1 runs the rest (ew_spmv.cu, layout_spmv).
    int64_t head_warps = 0;
    std::shared_ptr<SideStream> side;
    bool imported = false;  // built elsewhere: K2 may not cover every row
    DevBuf<double> values;
    // int32 columns per slot. After shrink_columns (compact or grouped
    // layouts, whose kernels read the 16-bit / grouped forms) only the wide
    // warps' columns stay, slot s of wide warp w at cols[col_shift[w] + s]
    // (col_shift empty and cols empty: a grouped int32 layout); cols_full
    // false then, and decode_columns rebuilds the whole slab on demand.
    DevBuf<int32_t> cols;
    DevBuf<int64_t> col_shift;
    bool cols_full = true;
    DevBuf<int64_t> warp_offset;
    DevBuf<int32_t> maxrows, rows_in_warp, reduction, rows_offset_warp;
    DevBuf<int32_t> fwd, inv, slen;
    // K1 with every warp's columns inside 0xFFFF of each other: the kernels
    // stream 16-bit offsets from the warp's smallest column instead of the
    // int32 columns (which stay for export / refresh maps)
    int compact = 0;
    int64_t narrow_slots = 0;  // slots outside the wide (int32) warps
    DevBuf<uint16_t> cols16;   // per slot: col - col_base[w], 0xFFFF = padding (column 0)
    DevBuf<int32_t> col_base;  // per warp
    // Grouped columns (K1 over 64 MB, ws = 32): consecutive lanes of a layout
    // warp with identical column lists (the 3 unknowns of a node in a
    // 3-DOF mesh) share one stored list; a lane reads its step-j column at
    // gcols[goff[w] + j * ngrp[w] + lane_grp[p]] (16-bit offsets from
    // col_base[w] when the layout is compact, else int32). The int32 / 16-bit
    // slabs stay (export, refresh maps, the staged host pipeline).
    int grouped = 0;
    int64_t grouped_slots = 0;   // stored grouped column entries
    int64_t grouped_col_bytes = 0;  // column bytes a grouped SpMV launch streams
    DevBuf<uint8_t> lane_grp;    // per sorted row
    DevBuf<uint8_t> ngrp;        // per warp
    DevBuf<int64_t> goff;        // per warp
    DevBuf<int32_t> gcols;       // int32 form
    DevBuf<uint16_t> gcols16;    // compact form
    DevBuf<int64_t> slot_map;  // lazily built value_slot_map (export)
    DevBuf<int64_t> src_map;   // lazily built per-slot source entry (values-only refresh)
    size_t device_bytes() const {
        return values.bytes() + cols.bytes() + warp_offset.bytes() + maxrows.bytes() +
               rows_in_warp.bytes() + reduction.bytes() + rows_offset_warp.bytes() + fwd.bytes() +
               inv.bytes() + slen.bytes() + slot_map.bytes() + src_map.bytes() + cols16.bytes() + col_base.bytes() +
               lane_grp.bytes() + ngrp.bytes() + goff.bytes() + gcols.bytes() + gcols16.bytes() +
               col_shift.bytes();
    }
};

// The paper's comparison formats (formats.hpp:11-53): csr_vector and coo run
// on the CSR arrays, ell / hyb on their own padded column-major slabs.
struct FormatData {
    enum Kind { kCsrVector, kCoo, kEll, kHyb } kind = kCsrVector;
    int32_t ws = 32;
    int64_t nrows = 0, ncols = 0, width = 0, k_ell = 0, coo_nnz = 0, stored_slots = 0;
    const CsrData* csr = nullptr;
    DevBuf<double> ell_v;
    DevBuf<int32_t> ell_c;
    DevBuf<int32_t> coo_rows, coo_cols;  // coo: rows only (cols/vals are the CSR's)
    DevBuf<double> coo_vals;
    size_t device_bytes() const {
        return ell_v.bytes() + ell_c.bytes() + coo_rows.bytes() + coo_cols.bytes() + coo_vals.bytes();
    }
};

namespace cg {
struct State;
}

// Device CG working set, kept between solves: buffers, the pinned polling
// slots and the CUDA graph of one block of iterations. Reused, a solve does
// no cudaMalloc / cudaFree / cudaMallocHost (which synchronise the device and
// can stall it for milliseconds) and no graph capture.
struct CgWorkspace {
    std::mutex mu;  // one solve at a time; a concurrent solve gets its own
    int64_t n = -1;
    DevBuf<double> r, p, q, x, b, diag, hist, partials;
    DevBuf<unsigned> tickets;
    DevBuf<cg::State> st;
    void* hst = nullptr;  // pinned cg::State[2]
    cudaEvent_t ev[2] = {nullptr, nullptr};
    cudaStream_t cap = nullptr;
    cudaGraphExec_t exec = nullptr;
    int64_t per_block = 0;  // launches per graph replay (accounting)
    // what the graph was captured with
    double g_tol = 0.0, g_div = 0.0;
    int64_t g_interval = -1, g_hist = -1;
    int g_jacobi = -1;
    CgWorkspace() = default;
    CgWorkspace(const CgWorkspace&) = delete;
    CgWorkspace& operator=(const CgWorkspace&) = delete;
    ~CgWorkspace() {
        if (exec) cudaGraphExecDestroy(exec);
        if (cap) cudaStreamDestroy(cap);
        if (ev[0]) cudaEventDestroy(ev[0]);
        if (ev[1]) cudaEventDestroy(ev[1]);
        if (hst) cudaFreeHost(hst);
    }
};

// Host-buffer apply of a large K1 kernel as a copy / compute pipeline over
// the kernel's own layout (no second copy of the matrix): x goes up in B
// column chunks; the layout's warps run in B stages, stage b holding every
// warp whose rows all lie in row blocks <= b (chunk c's columns cover every
// column the rows of blocks <= c reference, so stage b needs chunks <= b).
// Row block b goes down after stage ystage[b] (usually b) while later stages
// compute (PCIe is full duplex); the few rows of a block whose warp runs
// later than that ("stragglers": e.g. mesh edge rows sharing a warp with rows
// of every block) are gathered after the last stage and written into y on
// the host. Same warps, lanes and padding as one whole-layout launch: the
// same y, bit for bit, for any x.
struct HostPipeline {
    int nstages = 0;
    std::vector<int64_t> c0;       // x chunk bounds, nstages + 1
    std::vector<int64_t> r0;       // row block bounds, nstages + 1
    std::vector<int> ystage;       // per row block: the stage after which it goes down
    std::vector<int64_t> wstart;   // stage b runs widx[wstart[b], wstart[b + 1])
    DevBuf<int32_t> widx;          // layout warps in stage order
    std::vector<int32_t> late;     // straggler rows (ascending)
    DevBuf<int32_t> late_d;
    DevBuf<double> late_y;
    double* late_h = nullptr;      // pinned
    DevBuf<double> x, y;
    cudaStream_t up = nullptr, down = nullptr;
    std::vector<cudaEvent_t> ev_x, ev_y;
    cudaEvent_t ev_start = nullptr, ev_done = nullptr;
    HostPipeline() = default;
    HostPipeline(const HostPipeline&) = delete;
    HostPipeline& operator=(const HostPipeline&) = delete;
    ~HostPipeline() {
        for (auto e : ev_x) cudaEventDestroy(e);
        for (auto e : ev_y) cudaEventDestroy(e);
        if (ev_start) cudaEventDestroy(ev_start);
        if (ev_done) cudaEventDestroy(ev_done);
        if (up) cudaStreamDestroy(up);
        if (down) cudaStreamDestroy(down);
        if (late_h) cudaFreeHost(late_h);
    }
};

struct KernelData {
    std::string id;
    int64_t nrows = 0, ncols = 0, nnz = 0, stored_slots = 0;
    bool reordered = false;  // r / rs variants: perm set, apply permutes in/out
    bool locality = false;   // EW_ROW_ORDER_LOCALITY: perm is the locality order
    std::shared_ptr<CsrData> csr;        // csr_ref, and the arrays of csr_vector / coo
    std::shared_ptr<LayoutData> layout;  // k1* / k2*
    std::shared_ptr<FormatData> format;  // csr_vector / coo / ell / hyb
    DevBuf<int64_t> entry_dst;           // r / rs: original entry -> reordered entry (refresh)
    // CG working sets for cg_solve (0) and cg_solve_permuted (1)
    mutable CgWorkspace cg_ws[2];
    // host-buffer apply pipeline (built on first use; holds a stage plan of
    // the layout's warps and staging vectors, no matrix values)
    mutable std::mutex pipe_mu;
    mutable std::unique_ptr<HostPipeline> pipe;
};

// y = A x with x, y in host memory through the kernel's HostPipeline; false
// when the kernel does not qualify (not a large plain K1) or is busy.
bool kernel_apply_host(const KernelData& k, const double* x, double* y, cudaStream_t s);

std::shared_ptr<FormatData> build_format(const CsrData& m, const std::string& id, int32_t ws, int64_t hyb_k_ell,
                                         cudaStream_t s);
void format_spmv(const FormatData& f, const CsrData& m, const double* x, double* y, cudaStream_t s,
                 const int* done);
int64_t hyb_default_k_ell(const CsrData& m, cudaStream_t s);

// ---- internal API across translation units ---------------------------------
void validate_config(const ew_warp_config& c);
std::shared_ptr<CsrData> csr_upload(int64_t nrows, int64_t ncols, int64_t n_ro, const int64_t* ro,
                                    int64_t nnz, const int64_t* ci, const double* v,
                                    ew_mem_kind mem, bool canonical, cudaStream_t s);
void csr_spmv(const CsrData& m, const double* x, double* y, cudaStream_t s);
std::shared_ptr<CsrData> csr_clone(const CsrData& m, cudaStream_t s);
void csr_diagonal(const CsrData& m, double* d, cudaStream_t s);
void sort_rows_desc(const CsrData& m, int32_t* fwd, int32_t* inv, int32_t* slen,
                    cudaStream_t s, unsigned long long* n_active_counter);
// make_reordered_r / make_reordered_rs (reorder.cpp:8-43): renumber columns
// by a permutation (fwd_in, host, nullable = sort_rows_desc) and/or sort each
// row's (column, value) pairs by column.
// dst_of (nullable) receives, per input entry, its index in the output.
std::shared_ptr<CsrData> reorder(const CsrData& m, const int64_t* fwd_in, bool renumber,
                                 bool sort_within_rows, int32_t* fwd_out, cudaStream_t s,
                                 DevBuf<int64_t>* dst_of = nullptr);
// Locality row order (ew_order.cu): a Cuthill-McKee BFS order of m's rows,
// and the operand of a locality-ordered r / rs kernel: op (reorder() output,
// P-numbered columns, m's row offsets) with its rows permuted into
// qf = stable longest-first sort of that order and columns renumbered to qi.
void locality_order(const CsrData& m, int32_t* order, cudaStream_t s);
std::shared_ptr<CsrData> locality_operand(const CsrData& m, const CsrData& op, const int32_t* pf, int32_t* qf,
                                          int32_t* qi, cudaStream_t s);
void layout_refresh_values_reordered(LayoutData& l, const CsrData& m, const int64_t* dst_of, cudaStream_t s);
// out[slot] = source entry of m for every slot of l (-1 for padding), mapped
// through orig_of when given.
void layout_src_map(const LayoutData& l, const CsrData& m, const int64_t* orig_of, int64_t* out, cudaStream_t s);

// ---- FEM assembly as K1 row sums (ew_assembly.cu) ----
struct AssemblyData {
    int64_t nelements = 0, nnodes = 0, nnz = 0;
    CsrData pattern;  // global tangent sparsity (values zero), diagonal included
    std::shared_ptr<LayoutData> tangent, residual;  // K1 layouts over contribution rows
    DevBuf<int64_t> tangent_src, residual_src;      // per slot: element-output index or -1
};
std::shared_ptr<AssemblyData> assembly_create(int64_t ne, const int64_t* elements_host, int64_t nnodes,
                                              const ew_warp_config& cfg, cudaStream_t s);
void assembly_pattern(const AssemblyData& A, int64_t* ro, int64_t* ci);
int64_t assembly_nnz(const AssemblyData& A);
void assembly_run(const AssemblyData& A, const double* ke, const double* re, double* tangent, const int64_t* dest,
                  double* residual, cudaStream_t s);
void assembly_run_into(const AssemblyData& A, const double* ke, const double* re, KernelData& k, double* residual,
                       cudaStream_t s);
std::shared_ptr<LayoutData> build_layout(const CsrData& m, int kind, const ew_warp_config& cfg,
                                         int64_t threshold, bool sort_rows, bool row_major,
                                         cudaStream_t s);
std::shared_ptr<LayoutData> import_layout(const ew_layout_desc& d, cudaStream_t s);
// Where a CG-fused SpMV puts its p.q reduction (ew_spmv.cu k1_dot_kernel).
namespace cg {
struct State;
}
struct DotSink {
    double* partials;   // cg::dot_partials(SpMV CTAs)
    unsigned capacity;  // partials' length; a larger grid falls back to the dot kernel
    unsigned* tickets;  // cg::dot_tickets(SpMV CTAs) zeroed counters
    cg::State* st;      // decision / partition total
    int dist;           // 1: store the partition total in st->loc[slot]
    int slot = 0;       // DIST: 0 (also clears loc[1]) or 1 (a second row set)
};
// K1 SpMV with p.q fused (x is p); false when the layout has no fused path.
bool layout_spmv_dot(const LayoutData& l, const double* x, double* y, bool scatter, cudaStream_t s,
                     const int* done, const DotSink& sink);
// done (nullable, device): the launch is a no-op once *done != 0 (CG overrun).
void layout_spmv(const LayoutData& l, const double* x, double* y, bool scatter, cudaStream_t s,
                 const int* done = nullptr);
// Sorted K1, scatter store, over the layout warps widx[0, nidx) only (device
// list): the host-buffer pipeline runs a layout in stages this way.
void layout_spmv_warps(const LayoutData& l, const int32_t* widx, int64_t nidx, const double* x, double* y,
                       cudaStream_t s);
// Column bytes one SpMV launch of the layout streams (int32 / 16-bit / grouped).
// Counted over the stored slots (maxrows x ws per warp): the alignment gaps
// between slabs are never read.
inline int64_t layout_col_stream_bytes(const LayoutData& l) {
    if (l.grouped) return l.grouped_col_bytes;
    if (l.compact) return 2 * l.narrow_slots + 4 * (l.stored_slots - l.narrow_slots);
    return 4 * l.stored_slots;
}
// K1 with x split: columns [0, nown) from x, the rest from xg (scatter store).
void layout_spmv_split(const LayoutData& l, const double* x, const double* xg, int64_t nown, double* y,
                       cudaStream_t s);
void layout_build_slot_map(LayoutData& l, const CsrData& m, cudaStream_t s);
void layout_refresh_values(LayoutData& l, const CsrData& m, cudaStream_t s);
int64_t compute_k2_lanes(int64_t nnz_row, int64_t threshold, int64_t warp_size);
void gather(const int32_t* idx, const double* in, double* out, int64_t n, cudaStream_t s);
void scatter(const int32_t* idx, const double* in, double* out, int64_t n, cudaStream_t s);

// prepare_kernel (kernels.cpp:59-125) on device data.
std::shared_ptr<KernelData> prepare(const std::string& id, const CsrData& m, const ew_warp_config& c,
                                    const ew_kernel_options& o, cudaStream_t s);

// Kernel-level operator: y = A x in the kernel's "apply" (original) or
// "apply_permuted" (sorted) numbering; device pointers.
void kernel_apply(const KernelData& k, const double* x, double* y, bool permuted,
                  cudaStream_t s, const int* done = nullptr);
void csr_spmv_guarded(const CsrData& m, const double* x, double* y, cudaStream_t s, const int* done);

struct CgOutputs {
    ew_cg_result res{};
    std::vector<double> history;
    ew_status status = EW_OK;
    std::string message;
};
// The CG operator: y = A x on device pointers, enqueued on s. A host-callback
// operator (the reference's arbitrary SpmvFn closure) runs synchronously on
// the host thread; the solver then checks its done flag before each call.
bool kernel_apply_dot(const KernelData& k, const double* x, double* y, bool permuted, cudaStream_t s,
                      const int* done, const DotSink& sink);

struct CgOperator {
    virtual ~CgOperator() = default;
    virtual void apply(const double* x, double* y, cudaStream_t s, const int* done) const = 0;
    // y = A x with p.q = x.y reduced into `sink`; false: not fused, use apply + a dot kernel
    virtual bool apply_dot(const double*, double*, cudaStream_t, const int*, const DotSink&) const { return false; }
    virtual bool host_callback() const { return false; }
    virtual int64_t size() const = 0;
    // a working set kept between solves with this operator (nullable)
    virtual CgWorkspace* workspace() const { return nullptr; }
    // threads of the operator's SpMV launch (sizes the fused p.q partials)
    virtual int64_t spmv_threads() const { return size(); }
};
struct KernelOperator final : CgOperator {
    const KernelData& k;
    bool permuted;
    KernelOperator(const KernelData& kd, bool p) : k(kd), permuted(p) {}
    void apply(const double* x, double* y, cudaStream_t s, const int* done) const override {
        kernel_apply(k, x, y, permuted, s, done);
    }
    bool apply_dot(const double* x, double* y, cudaStream_t s, const int* done, const DotSink& sink) const override {
        return kernel_apply_dot(k, x, y, permuted, s, done, sink);
    }
    int64_t size() const override { return k.nrows == k.ncols ? k.nrows : -1; }
    CgWorkspace* workspace() const override { return &k.cg_ws[permuted ? 1 : 0]; }
    int64_t spmv_threads() const override {
        if (k.layout && k.layout->kind == EW_LAYOUT_K2) return std::max(k.nrows, k.layout->nwarps * k.layout->ws);
        return k.nrows;
    }
};
// Device CG. b, diag, x are device pointers in the operator's numbering.
CgOutputs cg_device(const CgOperator& op, const double* b, const double* diag, int64_t n,
                    const ew_cg_config& cfg, double* x, cudaStream_t s);
// ---- row-partitioned operator / CG (ew_dist.cu) ----
struct DistData;
std::vector<int64_t> partition_rows(const int64_t* ro, int64_t nrows, int32_t nparts);
std::shared_ptr<DistData> dist_create(int64_t nrows, int64_t ncols, const int64_t* ro, const int64_t* ci,
                                      const double* v, const int64_t* bounds, int32_t nparts, int32_t first,
                                      int32_t nlocal, const void* nccl_id, const std::string& kid,
                                      const ew_warp_config& cfg, const ew_kernel_options& opts, cudaStream_t s,
                                      bool peer = false);
// One partition per process over CUDA IPC (peer transport); setup data goes
// through the caller's allgather (ew_allgather_fn).
std::shared_ptr<DistData> dist_create_block_ipc(int64_t nglobal, const int64_t* bro, const int64_t* bci,
                                                const double* bv, const int64_t* bounds, int32_t nparts,
                                                int32_t rank, ew_allgather_fn allgather, void* user,
                                                const std::string& kid, const ew_warp_config& cfg,
                                                const ew_kernel_options& opts, cudaStream_t s);
struct BlockPlan {
    std::vector<int64_t> ghosts;                // ascending global ids outside the block
    std::vector<int64_t> counts;                // [h * G + g]: h's ghosts owned by g
    std::vector<std::vector<int64_t>> needs;    // per peer: rows of this block it needs
};
BlockPlan block_plan(int64_t nloc, const int64_t* bro, const int64_t* bci, const std::vector<int64_t>& bounds,
                     int32_t rank, ew_allgather_fn allgather, void* user);
std::shared_ptr<DistData> dist_create_block(int64_t nglobal, const int64_t* bro, const int64_t* bci,
                                            const double* bv, const int64_t* bounds, int32_t nparts, int32_t rank,
                                            const void* nccl_id, const std::string& kid, const ew_warp_config& cfg,
                                            const ew_kernel_options& opts, cudaStream_t s);
int64_t dist_owned_rows(const DistData& D);
void dist_part_info(const DistData& D, int32_t i, int64_t* r0, int64_t* r1, int64_t* nghost, int64_t* nsend);
void dist_layout_bytes(const DistData& D, int32_t i, int64_t* slots, int64_t* bytes);
void dist_spmv(DistData& D, const double* x, double* y, cudaStream_t s);
// Throws if a peer-transport wait timed out (synchronises s).
void dist_check_peers(const DistData& D, cudaStream_t s);
CgOutputs dist_cg(DistData& D, const double* b, const double* diag, const ew_cg_config& cfg, double* x,
                  cudaStream_t s);
void nccl_unique_id(void* out);
// Single process, several GPUs: partition g of the square host CSR on
// devices[g] (NULL: device g), peers over peer access (ew_mgpu_*).
struct MgpuData;
std::shared_ptr<MgpuData> mgpu_create(int64_t n, const int64_t* ro, const int64_t* ci, const double* v,
                                      int32_t nparts, const int32_t* devices, const std::string& kid,
                                      const ew_warp_config& cfg, const ew_kernel_options& opts);
int64_t mgpu_rows(const MgpuData& M);
void mgpu_spmv(MgpuData& M, const double* x, double* y);
CgOutputs mgpu_cg(MgpuData& M, const double* b, const double* diag, const ew_cg_config& cfg, double* x);

// Final status -> exception or result (+ history copied back).
CgOutputs cg_outputs(int status, long long iterations, const ew_cg_config& cfg, const double* hist_dev);

constexpr int kBlock = 256;
inline unsigned grid_for(int64_t n, int block = kBlock) {
    const int64_t g = (n + block - 1) / block;
    return static_cast<unsigned>(g < 1 ? 1 : g);
}
inline int log2_exact(int64_t v) {
    int l = 0;
    while ((int64_t{1} << l) < v) ++l;
    return l;
}

}  // namespace ew

// Device CSR: upload + validate_csr, the csr_ref SpMV, extract_diagonal,
// permutation gather/scatter.
#include <cuda.h>

#include "ew_internal.cuh"

namespace ew {

std::atomic<int64_t> g_launches{0};

void retain_pool() {
    static std::atomic<uint64_t> done_mask{0};  // one bit per device ordinal (< 64)
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
    const uint64_t bit = uint64_t{1} << dev;
    if (done_mask.load(std::memory_order_relaxed) & bit) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        // keep up to 8 GB of freed scratch (every per-call buffer of the
        // hot paths); beyond that, transient setup buffers (e.g. the int64
        // column staging of a 100M-row upload) go back to the driver
        uint64_t keep = uint64_t{8} << 30;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    done_mask.fetch_or(bit, std::memory_order_relaxed);
}

void load_all_kernels() {
    static std::mutex mu;
    static uint64_t done_mask = 0;  // one bit per device ordinal (< 64)
    int dev = 0;
    EW_CUDA_CHECK(cudaGetDevice(&dev));
    const uint64_t bit = dev < 64 ? uint64_t{1} << dev : 0;
    std::lock_guard<std::mutex> lock(mu);
    if (done_mask & bit) return;
    // each translation unit is one library; loading one kernel of it by
    // handle (cuKernelGetFunction) loads it into the current context
    using GetLibrary = CUresult (*)(CUlibrary*, CUkernel);
    using KernelCount = CUresult (*)(unsigned*, CUlibrary);
    using Enumerate = CUresult (*)(CUkernel*, unsigned, CUlibrary);
    using GetFunction = CUresult (*)(CUfunction*, CUkernel);
    auto entry = [](const char* name) -> void* {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion(name, &p, 12050, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return nullptr;
        return p;
    };
    auto get_library = reinterpret_cast<GetLibrary>(entry("cuKernelGetLibrary"));
    auto kernel_count = reinterpret_cast<KernelCount>(entry("cuLibraryGetKernelCount"));
    auto enumerate = reinterpret_cast<Enumerate>(entry("cuLibraryEnumerateKernels"));
    auto get_function = reinterpret_cast<GetFunction>(entry("cuKernelGetFunction"));
    const void* anchors[] = {kernel_anchor_assembly(), kernel_anchor_dist(), kernel_anchor_formats(),
                             kernel_anchor_kernel(), kernel_anchor_layout(), kernel_anchor_order(),
                             kernel_anchor_spmv(), kernel_anchor_csr()};
    if (!(get_library && kernel_count && enumerate && get_function)) {
        // a driver before CUDA 12.5: load what can be named (the anchors);
        // CUDA_MODULE_LOADING=EAGER in the environment covers the rest
        cudaFuncAttributes fa;
        for (const void* anchor : anchors) EW_CUDA_CHECK(cudaFuncGetAttributes(&fa, anchor));
        done_mask |= bit;
        return;
    }
    for (const void* anchor : anchors) {
        cudaKernel_t k = nullptr;
        EW_CUDA_CHECK(cudaGetKernel(&k, anchor));
        CUlibrary lib = nullptr;
        unsigned n = 0;
        require(get_library(&lib, reinterpret_cast<CUkernel>(k)) == CUDA_SUCCESS &&
                    kernel_count(&n, lib) == CUDA_SUCCESS,
                "load_all_kernels: cannot enumerate a kernel library");
        std::vector<CUkernel> all(n);
        require(n == 0 || enumerate(all.data(), n, lib) == CUDA_SUCCESS, "load_all_kernels: enumeration failed");
        for (CUkernel kk : all) {
            CUfunction fn = nullptr;
            require(get_function(&fn, kk) == CUDA_SUCCESS, "load_all_kernels: cannot load a kernel");
        }
    }
    done_mask |= bit;
}

namespace {

enum : int { kBadOrder = 1, kBadColumn = 2, kNotIncreasing = 4 };

// validate_csr (csr.cpp:57-73) for one row per thread, plus int64 -> int32
// column narrowing and the max row length. Flags OR into *err.
__global__ void validate_rows_kernel(const int64_t* __restrict__ ro, const int64_t* __restrict__ ci64,
                                     int32_t* __restrict__ ci32, int64_t nrows, int64_t ncols,
                                     int64_t nnz, int* err, int* maxrow) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= nrows) return;
    const int64_t lo = ro[r], hi = ro[r + 1];
    if (lo > hi || lo < 0 || hi > nnz) {
        atomicOr(err, kBadOrder);
        return;
    }
    int64_t prev = -1;
    int f = 0;
    for (int64_t k = lo; k < hi; ++k) {
        const int64_t c = ci64[k];
        if (c < 0 || c >= ncols) f |= kBadColumn;
        if (k > lo && prev >= c) f |= kNotIncreasing;
        prev = c;
        ci32[k] = static_cast<int32_t>(c);
    }
    if (f) atomicOr(err, f);
    const int64_t len = hi - lo;
    atomicMax(maxrow, static_cast<int>(len > 0x7fffffff ? 0x7fffffff : len));
}

// spmv_csr_reference (csr.cpp:75-86): one thread per row, sequential sum
// from 0.0 in CSR order; mul and add rounded separately (no FMA), so the
// result is bit-identical to the reference.
__global__ void csr_scalar_kernel(const int64_t* __restrict__ ro, const int32_t* __restrict__ ci,
                                  const double* __restrict__ v, const double* __restrict__ x,
                                  double* __restrict__ y, int64_t nrows, const int* done) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= nrows || (done && *done)) return;
    double sum = 0.0;
    for (int64_t k = ro[r], e = ro[r + 1]; k < e; ++k) sum = __dadd_rn(sum, __dmul_rn(v[k], x[ci[k]]));
    y[r] = sum;
}

// extract_diagonal (csr.cpp:106-117)
__global__ void diagonal_kernel(const int64_t* __restrict__ ro, const int32_t* __restrict__ ci,
                                const double* __restrict__ v, double* __restrict__ d,
                                int64_t nrows, int64_t ncols) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= nrows) return;
    double out = 0.0;
    if (r < ncols) {
        for (int64_t k = ro[r], e = ro[r + 1]; k < e; ++k) {
            if (ci[k] == r) {
                out = v[k];
                break;
            }
        }
    }
    d[r] = out;
}

__global__ void gather_kernel(const int32_t* __restrict__ idx, const double* __restrict__ in,
                              double* __restrict__ out, int64_t n) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n) out[k] = in[idx[k]];
}

__global__ void scatter_kernel(const int32_t* __restrict__ idx, const double* __restrict__ in,
                               double* __restrict__ out, int64_t n) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n) out[idx[k]] = in[k];
}

}  // namespace

std::shared_ptr<CsrData> csr_upload(int64_t nrows, int64_t ncols, int64_t n_ro, const int64_t* ro,
                                    int64_t nnz, const int64_t* ci, const double* v,
                                    ew_mem_kind mem, bool canonical, cudaStream_t s) {
    require(nrows >= 0 && ncols >= 0, "negative dimensions");
    require(n_ro == nrows + 1, "row_offsets length");
    require(nnz >= 0, "values/col_indices length mismatch");
    if (nrows > 0x7fffffff || ncols > 0x7fffffff)
        throw Error(EW_UNSUPPORTED, "device path supports at most 2^31-1 rows and columns");
    require(ro != nullptr, "row_offsets is null");
    require(nnz == 0 || (ci != nullptr && v != nullptr), "col_indices/values are null");
    auto m = std::make_shared<CsrData>();
    m->nrows = nrows;
    m->ncols = ncols;
    m->nnz = nnz;
    m->ro.alloc(nrows + 1);
    m->ci.alloc(nnz);
    m->v.alloc(nnz);
    const auto kind = mem == EW_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    EW_CUDA_CHECK(cudaMemcpyAsync(m->ro.get(), ro, (nrows + 1) * sizeof(int64_t), kind, s));
    if (nnz) EW_CUDA_CHECK(cudaMemcpyAsync(m->v.get(), v, nnz * sizeof(double), kind, s));
    int64_t ends[2] = {0, 0};
    EW_CUDA_CHECK(cudaMemcpyAsync(&ends[0], m->ro.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    EW_CUDA_CHECK(cudaMemcpyAsync(&ends[1], m->ro.get() + nrows, sizeof(int64_t),
                                  cudaMemcpyDeviceToHost, s));
    EW_CUDA_CHECK(cudaStreamSynchronize(s));
    require(ends[0] == 0, "row_offsets[0] != 0");
    require(ends[1] == nnz, "row_offsets[nrows] != nnz");

    Scratch<int64_t> ci64(nnz, s);
    if (nnz) EW_CUDA_CHECK(cudaMemcpyAsync(ci64.get(), ci, nnz * sizeof(int64_t), kind, s));
    Scratch<int> flags(2, s);
    EW_CUDA_CHECK(cudaMemsetAsync(flags.get(), 0, 2 * sizeof(int), s));
    if (nrows) {
        validate_rows_kernel<<<grid_for(nrows), kBlock, 0, s>>>(m->ro.get(), ci64.get(), m->ci.get(),
                                                                nrows, ncols, nnz, flags.get(),
                                                                flags.get() + 1);
        launched("validate_rows_kernel");
    }
    int h[2];
    EW_CUDA_CHECK(cudaMemcpyAsync(h, flags.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
    EW_CUDA_CHECK(cudaStreamSynchronize(s));
    require(!(h[0] & kBadOrder), "row_offsets not nondecreasing");
    require(!(h[0] & kBadColumn), "column out of range");
    require(!canonical || !(h[0] & kNotIncreasing), "columns not strictly increasing within row");
    m->maxrow = h[1];
    return m;
}

std::shared_ptr<CsrData> csr_clone(const CsrData& m, cudaStream_t s) {
    // prepared kernels own their matrix, as the reference's closures own a
    // copy (kernels.cpp:65-68): later updates of the caller's handle do not
    // reach an already prepared kernel
    auto c = std::make_shared<CsrData>();
    c->nrows = m.nrows;
    c->ncols = m.ncols;
    c->nnz = m.nnz;
    c->maxrow = m.maxrow;
    c->ro.alloc(m.nrows + 1);
    c->ci.alloc(m.nnz);
    c->v.alloc(m.nnz);
    EW_CUDA_CHECK(cudaMemcpyAsync(c->ro.get(), m.ro.get(), c->ro.bytes(), cudaMemcpyDeviceToDevice, s));
    if (m.nnz) {
        EW_CUDA_CHECK(cudaMemcpyAsync(c->ci.get(), m.ci.get(), c->ci.bytes(), cudaMemcpyDeviceToDevice, s));
        EW_CUDA_CHECK(cudaMemcpyAsync(c->v.get(), m.v.get(), c->v.bytes(), cudaMemcpyDeviceToDevice, s));
    }
    return c;
}

void csr_spmv_guarded(const CsrData& m, const double* x, double* y, cudaStream_t s, const int* done) {
    if (m.nrows == 0) return;
    csr_scalar_kernel<<<grid_for(m.nrows), kBlock, 0, s>>>(m.ro.get(), m.ci.get(), m.v.get(), x, y,
                                                           m.nrows, done);
    launched("csr_scalar_kernel");
}

void csr_spmv(const CsrData& m, const double* x, double* y, cudaStream_t s) {
    csr_spmv_guarded(m, x, y, s, nullptr);
}

void csr_diagonal(const CsrData& m, double* d, cudaStream_t s) {
    if (m.nrows == 0) return;
    diagonal_kernel<<<grid_for(m.nrows), kBlock, 0, s>>>(m.ro.get(), m.ci.get(), m.v.get(), d,
                                                         m.nrows, m.ncols);
    launched("diagonal_kernel");
}

void gather(const int32_t* idx, const double* in, double* out, int64_t n, cudaStream_t s) {
    if (n == 0) return;
    gather_kernel<<<grid_for(n), kBlock, 0, s>>>(idx, in, out, n);
    launched("gather_kernel");
}

void scatter(const int32_t* idx, const double* in, double* out, int64_t n, cudaStream_t s) {
    if (n == 0) return;
    scatter_kernel<<<grid_for(n), kBlock, 0, s>>>(idx, in, out, n);
    launched("scatter_kernel");
}

const void* kernel_anchor_csr() { return reinterpret_cast<const void*>(&validate_rows_kernel); }

}  // namespace ew

// Race-free FEM assembly as K1 row sums (reference
// fem/assembly.cpp:38-159): one contribution row per
// global tangent nonzero (and one per node for the residual), each listing
// the element-local entries that add into it in element-major order; rows
// packed into a K1 layout; per assembly the row sums run with the all-ones
// multiply elided.
//
// B200 form: the map is built on the device (stable radix sort of the 16 ne
// (row, col) keys -> pattern, run lengths -> contribution rows -> K1 layout
// -> per-slot source index). Per assembly ONE kernel gathers the element
// outputs through the source map and sums each contribution row in slot
// order, so there is no scatter pass and no flat staging array; the sums
// are bit-identical to the reference's scatter-then-row-sum (same addends,
// same order, padding slots adding 0.0). The tangent can be written straight
// into a prepared K1 kernel's slot order (the paper's "assemble into the
// format, skip the reorder").
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_run_length_encode.cuh>
#include <cub/device/device_scan.cuh>

#include "ew_internal.cuh"

namespace ew {

namespace {

__global__ void pair_keys_kernel(const int64_t* __restrict__ elem, int64_t ne, int64_t nnodes,
                                 uint64_t* __restrict__ tkeys, int64_t* __restrict__ tvals,
                                 uint64_t* __restrict__ rkeys, int64_t* __restrict__ rvals, int* bad) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= ne) return;
    int64_t t[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        t[i] = elem[4 * e + i];
        if (t[i] < 0 || t[i] >= nnodes) {
            atomicOr(bad, 1);
            t[i] = 0;
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        rkeys[4 * e + i] = static_cast<uint64_t>(t[i]);
        rvals[4 * e + i] = 4 * e + i;  // residual_slot enumeration (assembly.cpp:135-136)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            tkeys[16 * e + 4 * i + j] = static_cast<uint64_t>(t[i]) * static_cast<uint64_t>(nnodes) + t[j];
            tvals[16 * e + 4 * i + j] = 16 * e + 4 * i + j;  // tangent_slot enumeration (assembly.cpp:131-134)
        }
    }
}

// pattern columns and per-row counts from the unique (row, col) keys
__global__ void pattern_kernel(const uint64_t* __restrict__ ukeys, int64_t nnz, int64_t nnodes,
                               int32_t* __restrict__ ci, unsigned long long* __restrict__ row_count) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= nnz) return;
    const uint64_t key = ukeys[k];
    ci[k] = static_cast<int32_t>(key % static_cast<uint64_t>(nnodes));
    atomicAdd(row_count + key / static_cast<uint64_t>(nnodes), 1ull);
}

__global__ void count_nodes_kernel(const uint64_t* __restrict__ rkeys_sorted, int64_t n,
                                   unsigned long long* __restrict__ cnt) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n) atomicAdd(cnt + rkeys_sorted[k], 1ull);
}

__global__ void u64_to_i64_kernel(const unsigned long long* __restrict__ in, int64_t* __restrict__ out, int64_t n) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n) out[k] = static_cast<int64_t>(in[k]);
}

__global__ void i32_to_i64_kernel(const int32_t* __restrict__ in, int64_t* __restrict__ out, int64_t n) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n) out[k] = in[k];
}

// out[fwd[p]] = sum_j vals[src[slot(p, j)]] over the warp's maxrows steps
// (row_sum_kernel, assembly.cpp:38-74, with the flat staging array replaced
// by the source map). dest (nullable) redirects row r's sum to dest[r].
__global__ void __launch_bounds__(256) row_sum_gather_kernel(const int64_t* __restrict__ src,
                                                             const double* __restrict__ vals,
                                                             const int64_t* __restrict__ woff,
                                                             const int32_t* __restrict__ maxrows,
                                                             const int32_t* __restrict__ fwd, int64_t nrows,
                                                             int64_t n_active, int32_t ws, int32_t ws_log2,
                                                             const int64_t* __restrict__ dest, double* __restrict__ out) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= nrows || p >= n_active) return;  // empty contribution rows keep out = 0.0
    const int64_t w = p >> ws_log2;
    const int32_t mx = maxrows[w];
    int64_t s = woff[w] + (p & (ws - 1));
    double sum = 0.0;
    for (int32_t j = 0; j < mx; ++j, s += ws) {
        const int64_t k = src[s];
        sum = __dadd_rn(sum, k >= 0 ? vals[k] : 0.0);
    }
    const int64_t row = fwd[p];
    out[dest ? dest[row] : row] = sum;
}

std::shared_ptr<LayoutData> layout_over_counts(const int64_t* counts_dev, int64_t rows, int64_t total,
                                               const ew_warp_config& cfg, cudaStream_t s, CsrData& shape) {
    // a CSR that only carries row lengths (assembly.cpp:12-27)
    shape.nrows = rows;
    shape.ncols = 1;
    shape.nnz = total;
    shape.ro.alloc(rows + 1);
    shape.ci.alloc(total);
    shape.v.alloc(total);
    EW_CUDA_CHECK(cudaMemsetAsync(shape.ro.get(), 0, sizeof(int64_t), s));
    if (rows) {
        size_t bytes = 0;
        EW_CUDA_CHECK(cub::DeviceScan::InclusiveSum(nullptr, bytes, counts_dev, shape.ro.get() + 1, rows, s));
        Scratch<unsigned char> tmp(bytes, s);
        EW_CUDA_CHECK(cub::DeviceScan::InclusiveSum(tmp.get(), bytes, counts_dev, shape.ro.get() + 1, rows, s));
        launched("cub::DeviceScan::InclusiveSum");
    }
    if (total) {
        EW_CUDA_CHECK(cudaMemsetAsync(shape.ci.get(), 0, total * 4, s));
        EW_CUDA_CHECK(cudaMemsetAsync(shape.v.get(), 0, total * 8, s));
    }
    int64_t mx = 0;
    {
        // max row length for the sort keys
        std::vector<int64_t> h(static_cast<size_t>(rows));
        if (rows) EW_CUDA_CHECK(cudaMemcpyAsync(h.data(), counts_dev, rows * 8, cudaMemcpyDeviceToHost, s));
        EW_CUDA_CHECK(cudaStreamSynchronize(s));
        for (int64_t c : h) mx = std::max(mx, c);
    }
    shape.maxrow = static_cast<int32_t>(mx);
    return build_layout(shape, EW_LAYOUT_K1, cfg, 0, true, false, s);
}

template <typename K, typename V>
void radix_sort_pairs(K* keys, K* keys_out, V* vals, V* vals_out, int64_t n, int end_bit, cudaStream_t s) {
    size_t bytes = 0;
    EW_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys, keys_out, vals, vals_out, n, 0, end_bit, s));
    Scratch<unsigned char> tmp(bytes, s);
    EW_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, keys, keys_out, vals, vals_out, n, 0, end_bit, s));
    launched("cub::DeviceRadixSort::SortPairs");
}

}  // namespace

std::shared_ptr<AssemblyData> assembly_create(int64_t ne, const int64_t* elements_host, int64_t nnodes,
                                              const ew_warp_config& cfg, cudaStream_t s) {
    validate_config(cfg);
    require(ne >= 0 && nnodes >= 0, "assembly: negative sizes");
    require(nnodes < (int64_t{1} << 31), "assembly: at most 2^31-1 nodes");
    auto A = std::make_shared<AssemblyData>();
    A->nelements = ne;
    A->nnodes = nnodes;
    const int64_t nt = 16 * ne, nr = 4 * ne;
    Scratch<int64_t> elem(4 * ne, s);
    if (ne) EW_CUDA_CHECK(cudaMemcpyAsync(elem.get(), elements_host, 4 * ne * 8, cudaMemcpyHostToDevice, s));
    Scratch<uint64_t> tk(nt, s), tk2(nt, s), rk(nr, s), rk2(nr, s);
    Scratch<int64_t> tv(nt, s), tv2(nt, s), rv(nr, s), rv2(nr, s);
    Scratch<int> bad(1, s);
    EW_CUDA_CHECK(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
    if (ne) {
        pair_keys_kernel<<<grid_for(ne), kBlock, 0, s>>>(elem.get(), ne, nnodes, tk.get(), tv.get(), rk.get(),
                                                         rv.get(), bad.get());
        launched("pair_keys_kernel");
    }
    int hbad = 0;
    EW_CUDA_CHECK(cudaMemcpyAsync(&hbad, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    EW_CUDA_CHECK(cudaStreamSynchronize(s));
    require(!hbad, "assembly: element node index out of range");
    const uint64_t maxkey = static_cast<uint64_t>(nnodes) * static_cast<uint64_t>(nnodes);
    int bits_t = 1, bits_r = 1;
    while (bits_t < 64 && (uint64_t{1} << bits_t) < maxkey) ++bits_t;
    while (bits_r < 63 && (int64_t{1} << bits_r) < nnodes) ++bits_r;
    // stable: equal (row, col) keys keep the element-major enumeration order
    if (nt) radix_sort_pairs(tk.get(), tk2.get(), tv.get(), tv2.get(), nt, bits_t, s);
    if (nr) radix_sort_pairs(rk.get(), rk2.get(), rv.get(), rv2.get(), nr, bits_r, s);

    // pattern = unique keys; contribution row lengths = run lengths
    Scratch<uint64_t> ukeys(nt, s);
    Scratch<int32_t> runs(nt, s);
    Scratch<int64_t> nruns(1, s);
    int64_t nnz = 0;
    if (nt) {
        size_t bytes = 0;
        EW_CUDA_CHECK(cub::DeviceRunLengthEncode::Encode(nullptr, bytes, tk2.get(), ukeys.get(), runs.get(),
                                                         nruns.get(), nt, s));
        Scratch<unsigned char> tmp(bytes, s);
        EW_CUDA_CHECK(cub::DeviceRunLengthEncode::Encode(tmp.get(), bytes, tk2.get(), ukeys.get(), runs.get(),
                                                         nruns.get(), nt, s));
        launched("cub::DeviceRunLengthEncode::Encode");
        EW_CUDA_CHECK(cudaMemcpyAsync(&nnz, nruns.get(), 8, cudaMemcpyDeviceToHost, s));
        EW_CUDA_CHECK(cudaStreamSynchronize(s));
    }
    A->nnz = nnz;
    A->pattern.nrows = A->pattern.ncols = nnodes;
    A->pattern.nnz = nnz;
    A->pattern.ci.alloc(nnz);
    A->pattern.ro.alloc(nnodes + 1);
    A->pattern.v.alloc(nnz);
    if (nnz) EW_CUDA_CHECK(cudaMemsetAsync(A->pattern.v.get(), 0, nnz * 8, s));
    {
        Scratch<unsigned long long> rc(nnodes, s);
        if (nnodes) EW_CUDA_CHECK(cudaMemsetAsync(rc.get(), 0, nnodes * 8, s));
        if (nnz) {
            pattern_kernel<<<grid_for(nnz), kBlock, 0, s>>>(ukeys.get(), nnz, nnodes, A->pattern.ci.get(), rc.get());
            launched("pattern_kernel");
        }
        Scratch<int64_t> rc64(nnodes, s);
        if (nnodes) {
            u64_to_i64_kernel<<<grid_for(nnodes), kBlock, 0, s>>>(rc.get(), rc64.get(), nnodes);
            launched("u64_to_i64_kernel");
        }
        EW_CUDA_CHECK(cudaMemsetAsync(A->pattern.ro.get(), 0, 8, s));
        if (nnodes) {
            size_t bytes = 0;
            EW_CUDA_CHECK(cub::DeviceScan::InclusiveSum(nullptr, bytes, rc64.get(), A->pattern.ro.get() + 1, nnodes, s));
            Scratch<unsigned char> tmp(bytes, s);
            EW_CUDA_CHECK(
                cub::DeviceScan::InclusiveSum(tmp.get(), bytes, rc64.get(), A->pattern.ro.get() + 1, nnodes, s));
            launched("cub::DeviceScan::InclusiveSum");
        }
        EW_CUDA_CHECK(cudaStreamSynchronize(s));
    }
    // tangent contribution rows over pattern entries, residual rows over nodes
    {
        Scratch<int64_t> len(nnz, s);
        if (nnz) {
            i32_to_i64_kernel<<<grid_for(nnz), kBlock, 0, s>>>(runs.get(), len.get(), nnz);
            launched("i32_to_i64_kernel");
        }
        CsrData shape;
        A->tangent = layout_over_counts(len.get(), nnz, nt, cfg, s, shape);
        // the shape's entries are the sorted pairs: entry -> element-output index
        A->tangent_src.alloc(A->tangent->nslots);
        layout_src_map(*A->tangent, shape, tv2.get(), A->tangent_src.get(), s);
    }
    {
        Scratch<unsigned long long> cnt(nnodes, s);
        Scratch<int64_t> len(nnodes, s);
        if (nnodes) EW_CUDA_CHECK(cudaMemsetAsync(cnt.get(), 0, nnodes * 8, s));
        if (nr) {
            count_nodes_kernel<<<grid_for(nr), kBlock, 0, s>>>(rk2.get(), nr, cnt.get());
            launched("count_nodes_kernel");
        }
        if (nnodes) {
            u64_to_i64_kernel<<<grid_for(nnodes), kBlock, 0, s>>>(cnt.get(), len.get(), nnodes);
            launched("u64_to_i64_kernel");
        }
        CsrData shape;
        A->residual = layout_over_counts(len.get(), nnodes, nr, cfg, s, shape);
        A->residual_src.alloc(A->residual->nslots);
        layout_src_map(*A->residual, shape, rv2.get(), A->residual_src.get(), s);
    }
    EW_CUDA_CHECK(cudaStreamSynchronize(s));
    return A;
}

int64_t assembly_nnz(const AssemblyData& A) { return A.nnz; }

void assembly_pattern(const AssemblyData& A, int64_t* ro, int64_t* ci) {
    if (ro) EW_CUDA_CHECK(cudaMemcpy(ro, A.pattern.ro.get(), (A.nnodes + 1) * 8, cudaMemcpyDeviceToHost));
    if (ci && A.nnz) {
        std::vector<int32_t> h(static_cast<size_t>(A.nnz));
        EW_CUDA_CHECK(cudaMemcpy(h.data(), A.pattern.ci.get(), A.nnz * 4, cudaMemcpyDeviceToHost));
        for (int64_t k = 0; k < A.nnz; ++k) ci[k] = h[k];
    }
}

// Row sums into tangent (CSR value order, or through `dest` into a prepared
// kernel's slots) and residual. ke: ne x 16, re: ne x 4, device pointers.
namespace {
__global__ void compose_kernel(const int64_t* __restrict__ slot_map, const int64_t* __restrict__ entry_dst,
                               int64_t* __restrict__ out, int64_t n) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n) out[k] = slot_map[entry_dst ? entry_dst[k] : k];
}
}  // namespace

// Assemble the tangent straight into a prepared K1/K2 kernel's slot order
// (pattern entry k -> the slot its value occupies), residual as usual.
void assembly_run_into(const AssemblyData& A, const double* ke, const double* re, KernelData& k, double* residual,
                       cudaStream_t s) {
    require(k.layout && !k.format, "assembly: the kernel must be an ELL-WARP (k1 / k2 family) kernel");
    require(k.nrows == A.nnodes && k.nnz == A.nnz, "assembly: the kernel was not prepared on the assembly pattern");
    LayoutData& l = *k.layout;
    layout_build_slot_map(l, A.pattern, s);  // operand entry -> slot (r / rs keep the pattern's row offsets)
    Scratch<int64_t> dest(A.nnz, s);
    if (A.nnz) {
        compose_kernel<<<grid_for(A.nnz), kBlock, 0, s>>>(l.slot_map.get(), k.reordered ? k.entry_dst.get() : nullptr,
                                                          dest.get(), A.nnz);
        launched("compose_kernel");
    }
    assembly_run(A, ke, re, l.values.get(), dest.get(), residual, s);
}

void assembly_run(const AssemblyData& A, const double* ke, const double* re, double* tangent, const int64_t* dest,
                  double* residual, cudaStream_t s) {
    auto go = [&](const LayoutData& l, const int64_t* src, const double* vals, const int64_t* d, double* out,
                  int64_t nrows) {
        if (!nrows) return;
        if (!d) EW_CUDA_CHECK(cudaMemsetAsync(out, 0, nrows * 8, s));  // empty rows are 0.0 (assembly.cpp:41)
        row_sum_gather_kernel<<<grid_for(l.nrows), kBlock, 0, s>>>(src, vals, l.warp_offset.get(), l.maxrows.get(),
                                                                   l.fwd.get(), l.nrows, l.n_active, l.ws, l.ws_log2,
                                                                   d, out);
        launched("row_sum_gather_kernel");
    };
    if (tangent) go(*A.tangent, A.tangent_src.get(), ke, dest, tangent, A.nnz);
    if (residual) go(*A.residual, A.residual_src.get(), re, nullptr, residual, A.nnodes);
}

const void* kernel_anchor_assembly() { return reinterpret_cast<const void*>(&pair_keys_kernel); }

}  // namespace ew

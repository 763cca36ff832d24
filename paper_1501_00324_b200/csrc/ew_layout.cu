// Device construction of the ELL-WARP layouts (paper §ELL-WARP):
// stable longest-first row sort, K1 / K2 per-warp metadata, column-major fill,
// r / rs column renumbering, value_slot_map and the values-only refresh.
//
// Everything runs on the device; the host only sizes allocations. The
// reference builds the same arrays with sequential loops
// (warp_layout.cpp:32-147, permutation.cpp:49-55, reorder.cpp:8-43); parity
// is bit-exact on every array (tests/test_gpu_layout.py).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <cstdlib>

#include "ew_internal.cuh"

namespace ew {

namespace {

__device__ __forceinline__ int64_t ceil_div_d(int64_t a, int64_t b) { return (a + b - 1) / b; }

// compute_k2_lanes (warp_layout.cpp:76-84); arguments pre-validated.
__device__ __forceinline__ int32_t k2_lanes(int64_t len, int64_t t, int32_t ws) {
    if (len > int64_t(ws) * t) return ws;
    int32_t lanes = 1;
    while (ceil_div_d(len, lanes) > t) lanes <<= 1;
    return lanes;
}

__global__ void sort_keys_kernel(const int64_t* __restrict__ ro, uint32_t* __restrict__ keys,
                                 int32_t* __restrict__ ids, int64_t n, int32_t maxrow) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= n) return;
    // ascending radix sort on (maxrow - len) is a stable longest-first sort
    keys[r] = static_cast<uint32_t>(maxrow - static_cast<int32_t>(ro[r + 1] - ro[r]));
    ids[r] = static_cast<int32_t>(r);
}

__global__ void finish_perm_kernel(const int64_t* __restrict__ ro, const int32_t* __restrict__ fwd,
                                   int32_t* __restrict__ inv, int32_t* __restrict__ slen,
                                   int64_t n, unsigned long long* n_active) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int32_t row = fwd[p];
    inv[row] = static_cast<int32_t>(p);
    const int32_t len = static_cast<int32_t>(ro[row + 1] - ro[row]);
    slen[p] = len;
    if (len > 0) atomicAdd(n_active, 1ull);
}

__global__ void identity_perm_kernel(const int64_t* __restrict__ ro, int32_t* __restrict__ fwd,
                                     int32_t* __restrict__ inv, int32_t* __restrict__ slen,
                                     int64_t n, unsigned long long* n_active) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    fwd[p] = inv[p] = static_cast<int32_t>(p);
    const int32_t len = static_cast<int32_t>(ro[p + 1] - ro[p]);
    slen[p] = len;
    if (len > 0) atomicAdd(n_active, 1ull);
}

// K1 metadata (warp_layout.cpp:47-59): warp w holds sorted positions
// [w*ws, min(w*ws+ws, n)), padded to its longest row.
__global__ void k1_meta_kernel(const int32_t* __restrict__ slen, int64_t n, int32_t ws, int64_t nw,
                               int64_t unit, int32_t* __restrict__ maxrows,
                               int32_t* __restrict__ rows_in_warp, int64_t* __restrict__ sizes,
                               unsigned long long* stored) {
    const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (w >= nw) return;
    const int64_t lo = w * ws;
    const int64_t hi = lo + ws < n ? lo + ws : n;
    int32_t mx = 0;
    for (int64_t p = lo; p < hi; ++p) mx = max(mx, slen[p]);
    maxrows[w] = mx;
    rows_in_warp[w] = static_cast<int32_t>(hi - lo);
    const int64_t sz = int64_t(mx) * ws;
    sizes[w] = ceil_div_d(sz, unit) * unit;  // align_offset (warp_layout.cpp:12-16)
    atomicAdd(stored, static_cast<unsigned long long>(int64_t(mx) * (hi - lo)));
}

// K2 packing (warp_layout.cpp:99-120), step 1: lanes per sorted row and the
// start of each maximal run of equal lane counts (as an index to max-scan).
__global__ void k2_lanes_kernel(const int32_t* __restrict__ slen, int64_t n, int64_t t, int32_t ws,
                                int32_t* __restrict__ lanes, int64_t* __restrict__ run_mark) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int32_t l = k2_lanes(slen[p], t, ws);
    lanes[p] = l;
    const bool start = p == 0 || k2_lanes(slen[p - 1], t, ws) != l;
    run_mark[p] = start ? p : 0;
}

// step 2: a warp opens at each run start and every ws/lanes rows inside a
// run -- exactly where the greedy loop closes the previous warp.
__global__ void k2_warp_start_kernel(const int32_t* __restrict__ lanes,
                                     const int64_t* __restrict__ run_start, int64_t n, int32_t ws,
                                     int32_t* __restrict__ flag) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int64_t cap = ws / lanes[p];
    flag[p] = ((p - run_start[p]) % cap) == 0 ? 1 : 0;
}

// step 3: per-warp metadata from the inclusive scan of warp-start flags.
__global__ void k2_meta_kernel(const int32_t* __restrict__ flag, const int32_t* __restrict__ wid,
                               const int32_t* __restrict__ lanes, int64_t n,
                               int32_t* __restrict__ rows_offset_warp,
                               int32_t* __restrict__ reduction) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n || !flag[p]) return;
    const int32_t w = wid[p] - 1;
    rows_offset_warp[w] = static_cast<int32_t>(p);
    reduction[w] = lanes[p];
}

__global__ void k2_meta2_kernel(const int32_t* __restrict__ slen,
                                const int32_t* __restrict__ rows_offset_warp,
                                const int32_t* __restrict__ reduction, int64_t n, int64_t nw,
                                int32_t ws, int64_t unit, int32_t* __restrict__ rows_in_warp,
                                int32_t* __restrict__ maxrows, int64_t* __restrict__ sizes,
                                unsigned long long* stored, int* max_red) {
    const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (w >= nw) return;
    const int64_t lo = rows_offset_warp[w];
    const int64_t hi = w + 1 < nw ? rows_offset_warp[w + 1] : n;
    const int32_t red = reduction[w];
    int32_t mx = 0;
    for (int64_t p = lo; p < hi; ++p) mx = max(mx, static_cast<int32_t>(ceil_div_d(slen[p], red)));
    rows_in_warp[w] = static_cast<int32_t>(hi - lo);
    maxrows[w] = mx;
    const int64_t sz = int64_t(mx) * ws;
    sizes[w] = ceil_div_d(sz, unit) * unit;
    atomicAdd(stored, static_cast<unsigned long long>(int64_t(mx) * red * (hi - lo)));
    atomicMax(max_red, red);
}

// Source CSR entry of local slot `local` of warp w, or -1 for padding.
// K1: lane = local % ws, j = local / ws (column-major) or lane = local / mx,
// j = local % mx (row_major diagnostic). K2: lane = r*red + e/mx, j = e%mx
// (warp_layout.cpp:138-139) => r = lane/red, e = (lane%red)*mx + j.
struct SlotMapper {
    const int64_t* ro;
    const int32_t* fwd;
    const int32_t* slen;
    const int64_t* woff;
    const int32_t* maxrows;
    const int32_t* rows_in_warp;
    const int32_t* reduction;         // nullptr for K1
    const int32_t* rows_offset_warp;  // nullptr for K1
    int32_t ws, ws_log2, row_major;
    int64_t nwarps, nslots;

    __device__ __forceinline__ int64_t source(int64_t w, int64_t local, int32_t mx, int32_t red,
                                              int64_t first, int32_t nr) const {
        int64_t lane, j;
        if (row_major) {
            lane = local / mx;
            j = local - lane * mx;
        } else {
            j = local >> ws_log2;
            lane = local & (ws - 1);
        }
        const int64_t r = lane / red;
        const int64_t e = (lane - r * red) * mx + j;
        if (r >= nr) return -1;
        const int64_t pos = first + r;
        if (e >= slen[pos]) return -1;
        return ro[fwd[pos]] + e;
    }
};

// One hardware warp per layout warp (grid-stride): coalesced writes of the
// warp's slab, alignment gap zeroed so no separate memset pass is needed.
__global__ void fill_kernel(SlotMapper M, const double* __restrict__ v, const int32_t* __restrict__ ci,
                            double* __restrict__ out_v, int32_t* __restrict__ out_c) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nhw = (gridDim.x * (int64_t)blockDim.x) >> 5;
    for (int64_t w = gw; w < M.nwarps; w += nhw) {
        const int64_t off = M.woff[w];
        const int64_t end = w + 1 < M.nwarps ? M.woff[w + 1] : M.nslots;
        const int32_t mx = M.maxrows[w];
        const int32_t red = M.reduction ? M.reduction[w] : 1;
        const int64_t first = M.rows_offset_warp ? M.rows_offset_warp[w] : (w << M.ws_log2);
        const int32_t nr = M.rows_in_warp[w];
        const int64_t count = int64_t(mx) * M.ws;
        for (int64_t local = lane; local < end - off; local += 32) {
            const int64_t k = local < count ? M.source(w, local, mx, red, first, nr) : -1;
            out_v[off + local] = k >= 0 ? v[k] : 0.0;
            out_c[off + local] = k >= 0 ? ci[k] : 0;
        }
    }
}

// value_slot_map (warp_layout.cpp:149-174): CSR entry -> flat slot.
__global__ void slot_map_kernel(SlotMapper M, int64_t* __restrict__ map) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nhw = (gridDim.x * (int64_t)blockDim.x) >> 5;
    for (int64_t w = gw; w < M.nwarps; w += nhw) {
        const int64_t off = M.woff[w];
        const int32_t mx = M.maxrows[w];
        const int32_t red = M.reduction ? M.reduction[w] : 1;
        const int64_t first = M.rows_offset_warp ? M.rows_offset_warp[w] : (w << M.ws_log2);
        const int32_t nr = M.rows_in_warp[w];
        const int64_t count = int64_t(mx) * M.ws;
        for (int64_t local = lane; local < count; local += 32) {
            const int64_t k = M.source(w, local, mx, red, first, nr);
            if (k >= 0) map[k] = off + local;
        }
    }
}

// Per-slot source entry (-1 for padding and alignment gaps): the inverse of
// value_slot_map, so the values-only refresh is a gather with coalesced
// writes instead of a scatter through the slot map. orig_of (nullable) maps
// the layout's operand entries (an r / rs matrix) back to the original's.
__global__ void src_map_kernel(SlotMapper M, const int64_t* __restrict__ orig_of, int64_t* __restrict__ src) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nhw = (gridDim.x * (int64_t)blockDim.x) >> 5;
    for (int64_t w = gw; w < M.nwarps; w += nhw) {
        const int64_t off = M.woff[w];
        const int64_t end = w + 1 < M.nwarps ? M.woff[w + 1] : M.nslots;
        const int32_t mx = M.maxrows[w];
        const int32_t red = M.reduction ? M.reduction[w] : 1;
        const int64_t first = M.rows_offset_warp ? M.rows_offset_warp[w] : (w << M.ws_log2);
        const int32_t nr = M.rows_in_warp[w];
        const int64_t count = int64_t(mx) * M.ws;
        for (int64_t local = lane; local < end - off; local += 32) {
            int64_t k = local < count ? M.source(w, local, mx, red, first, nr) : -1;
            if (k >= 0 && orig_of) k = orig_of[k];
            src[off + local] = k;
        }
    }
}

__global__ void refresh_gather_kernel(const int64_t* __restrict__ src, const double* __restrict__ v,
                                      double* __restrict__ out, int64_t nslots) {
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= nslots) return;
    const int64_t k = src[s];
    if (k >= 0) out[s] = v[k];  // padding slots keep their 0.0
}

__global__ void invert_kernel(const int64_t* __restrict__ dst_of, int64_t* __restrict__ orig_of, int64_t n) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n) orig_of[dst_of[k]] = k;
}

// make_reordered_r (reorder.cpp:8-17): c -> inverse[c]
__global__ void renumber_kernel(const int32_t* __restrict__ ci, const int32_t* __restrict__ inv,
                                int32_t* __restrict__ out, int64_t nnz) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < nnz) out[k] = inv[ci[k]];
}

// make_reordered_rs (reorder.cpp:19-43): one warp per row; each entry's
// destination is its rank among the row's (distinct) renumbered columns.
__global__ void row_rank_sort_kernel(const int64_t* __restrict__ ro, const int32_t* __restrict__ c_in,
                                     const double* __restrict__ v_in, int32_t* __restrict__ c_out,
                                     double* __restrict__ v_out, int64_t* __restrict__ dst_of, int64_t nrows) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nhw = (gridDim.x * (int64_t)blockDim.x) >> 5;
    for (int64_t r = gw; r < nrows; r += nhw) {
        const int64_t lo = ro[r], hi = ro[r + 1];
        for (int64_t k = lo + lane; k < hi; k += 32) {
            const int32_t c = c_in[k];
            int64_t rank = 0;
            // stable rank; keys are distinct for a renumbered canonical row
            for (int64_t q = lo; q < hi; ++q) rank += (c_in[q] < c || (c_in[q] == c && q < k)) ? 1 : 0;
            c_out[lo + rank] = c;
            v_out[lo + rank] = v_in[k];
            if (dst_of) dst_of[k] = lo + rank;  // where entry k of the input went
        }
    }
}

__global__ void iota_kernel(int64_t* __restrict__ out, int64_t n) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n) out[k] = k;
}


// ---- compact (16-bit) columns for K1 ---------------------------------------
// One hardware warp per layout warp (grid-stride): the smallest and largest
// column over the warp's real entries (padding excluded).
__global__ void compact_range_kernel(const int32_t* __restrict__ cols, const int64_t* __restrict__ woff,
                                     const int32_t* __restrict__ maxrows, const int32_t* __restrict__ rows_in_warp,
                                     const int32_t* __restrict__ slen, int32_t ws, int32_t ws_log2, int64_t nwarps,
                                     int32_t* __restrict__ base, int64_t* fail) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nhw = (gridDim.x * (int64_t)blockDim.x) >> 5;
    for (int64_t w = gw; w < nwarps; w += nhw) {
        const int64_t n = int64_t(maxrows[w]) * ws, off = woff[w];
        const int32_t nr = rows_in_warp[w];
        int32_t mn = 0x7fffffff, mx = -1;
        for (int64_t i = lane; i < n; i += 32) {
            const int32_t l = static_cast<int32_t>(i & (ws - 1));
            const int64_t j = i >> ws_log2;
            if (l >= nr || j >= slen[w * ws + l]) continue;
            const int32_t c = cols[off + i];
            mn = min(mn, c);
            mx = max(mx, c);
        }
        mn = __reduce_min_sync(0xffffffffu, mn);
        mx = __reduce_max_sync(0xffffffffu, mx);
        if (lane == 0) {
            const bool wide = mx >= 0 && int64_t(mx) - mn >= 0xFFFF;
            base[w] = wide ? -1 : (mx < 0 ? 0 : mn);
            if (wide) atomicAdd(reinterpret_cast<unsigned long long*>(fail), static_cast<unsigned long long>(n));
        }
    }
}

__global__ void compact_encode_kernel(const int32_t* __restrict__ cols, const int64_t* __restrict__ woff,
                                      const int32_t* __restrict__ maxrows, const int32_t* __restrict__ rows_in_warp,
                                      const int32_t* __restrict__ slen, int32_t ws, int32_t ws_log2, int64_t nwarps,
                                      const int32_t* __restrict__ base, uint16_t* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nhw = (gridDim.x * (int64_t)blockDim.x) >> 5;
    for (int64_t w = gw; w < nwarps; w += nhw) {
        const int64_t n = int64_t(maxrows[w]) * ws, off = woff[w];
        const int32_t nr = rows_in_warp[w], b = base[w];
        if (b < 0) continue;  // stays on the int32 slab
        for (int64_t i = lane; i < n; i += 32) {
            const int32_t l = static_cast<int32_t>(i & (ws - 1));
            const int64_t j = i >> ws_log2;
            const bool valid = l < nr && j < slen[w * ws + l];
            out[off + i] = valid ? static_cast<uint16_t>(cols[off + i] - b) : uint16_t{0xFFFF};
        }
    }
}

unsigned fill_grid(int64_t nwarps) {
    // 8 hardware warps per CTA, enough CTAs to cover every SM several times.
    int64_t g = (nwarps + 7) / 8;
    if (g > 148 * 32) g = 148 * 32;
    return static_cast<unsigned>(g < 1 ? 1 : g);
}

void exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s) {
    size_t bytes = 0;
    EW_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, s));
    Scratch<unsigned char> tmp(bytes, s);
    EW_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, in, out, n, s));
    launched("cub::DeviceScan::ExclusiveSum");
}

template <typename T>
T read_scalar(const T* dptr, cudaStream_t s) {
    T h{};
    EW_CUDA_CHECK(cudaMemcpyAsync(&h, dptr, sizeof(T), cudaMemcpyDeviceToHost, s));
    EW_CUDA_CHECK(cudaStreamSynchronize(s));
    return h;
}

SlotMapper mapper_of(const LayoutData& l, const CsrData& m) {
    SlotMapper M;
    M.ro = m.ro.get();
    M.fwd = l.fwd.get();
    M.slen = l.slen.get();
    M.woff = l.warp_offset.get();
    M.maxrows = l.maxrows.get();
    M.rows_in_warp = l.rows_in_warp.get();
    M.reduction = l.kind == EW_LAYOUT_K2 ? l.reduction.get() : nullptr;
    M.rows_offset_warp = l.kind == EW_LAYOUT_K2 ? l.rows_offset_warp.get() : nullptr;
    M.ws = l.ws;
    M.ws_log2 = l.ws_log2;
    M.row_major = l.row_major;
    M.nwarps = l.nwarps;
    M.nslots = l.nslots;
    return M;
}

}  // namespace

void validate_config(const ew_warp_config& c) {
    // WarpModelConfig::validate (warp_model.cpp:7-14)
    require(c.warp_size > 0 && (c.warp_size & (c.warp_size - 1)) == 0,
            "warp_size must be a power of two");
    require(c.block_size >= c.warp_size && c.block_size % c.warp_size == 0,
            "block_size must be a positive multiple of warp_size");
    require(c.segment_bytes > 0 && (c.segment_bytes & (c.segment_bytes - 1)) == 0,
            "segment_bytes must be a power of two");
    require(c.cache_lines > 0, "cache_lines must be positive");
}

int64_t compute_k2_lanes(int64_t nnz_row, int64_t threshold, int64_t warp_size) {
    require(threshold >= 1, "compute_k2_lanes: threshold must be >= 1");
    require(warp_size >= 1 && (warp_size & (warp_size - 1)) == 0,
            "compute_k2_lanes: warp_size must be a power of two");
    if (nnz_row > warp_size * threshold) return warp_size;
    int64_t lanes = 1;
    while ((nnz_row + lanes - 1) / lanes > threshold) lanes <<= 1;
    return lanes;
}

void sort_rows_desc(const CsrData& m, int32_t* fwd, int32_t* inv, int32_t* slen, cudaStream_t s,
                    unsigned long long* n_active) {
    const int64_t n = m.nrows;
    if (n == 0) return;
    Scratch<uint32_t> keys(n, s), keys_out(n, s);
    Scratch<int32_t> ids(n, s);
    Scratch<unsigned long long> cnt(n_active ? 0 : 1, s);
    unsigned long long* counter = n_active ? n_active : cnt.get();
    sort_keys_kernel<<<grid_for(n), kBlock, 0, s>>>(m.ro.get(), keys.get(), ids.get(), n, m.maxrow);
    launched("sort_keys_kernel");
    const int end_bit = std::max(1, log2_exact(int64_t(m.maxrow) + 1));
    size_t bytes = 0;
    EW_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.get(), keys_out.get(), ids.get(),
                                                  fwd, n, 0, end_bit, s));
    Scratch<unsigned char> tmp(bytes, s);
    EW_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, keys.get(), keys_out.get(),
                                                  ids.get(), fwd, n, 0, end_bit, s));
    launched("cub::DeviceRadixSort::SortPairs");
    if (!n_active) EW_CUDA_CHECK(cudaMemsetAsync(counter, 0, sizeof(unsigned long long), s));
    finish_perm_kernel<<<grid_for(n), kBlock, 0, s>>>(m.ro.get(), fwd, inv, slen, n, counter);
    launched("finish_perm_kernel");
}

std::shared_ptr<CsrData> reorder(const CsrData& m, const int64_t* fwd_in, bool renumber,
                                 bool sort_within_rows, int32_t* fwd_out, cudaStream_t s, DevBuf<int64_t>* dst_of) {
    const int64_t n = m.nrows, nnz = m.nnz;
    if (dst_of) dst_of->alloc(nnz);
    Scratch<int32_t> fwd(renumber ? n : 0, s), inv(renumber ? n : 0, s), slen(renumber ? n : 0, s);
    if (renumber) {
        require(m.nrows == m.ncols, "make_reordered_r: matrix must be square");
        if (fwd_in) {
            // Permutation::from_forward (permutation.cpp:17-28) semantics
            std::vector<int32_t> hf(static_cast<size_t>(n)), hi(static_cast<size_t>(n), -1);
            for (int64_t k = 0; k < n; ++k) {
                const int64_t old = fwd_in[k];
                require(old >= 0 && old < n, "permutation index out of range");
                require(hi[old] == -1, "permutation not a bijection");
                hi[old] = static_cast<int32_t>(k);
                hf[k] = static_cast<int32_t>(old);
            }
            if (n) {
                EW_CUDA_CHECK(cudaMemcpyAsync(fwd.get(), hf.data(), n * 4, cudaMemcpyHostToDevice, s));
                EW_CUDA_CHECK(cudaMemcpyAsync(inv.get(), hi.data(), n * 4, cudaMemcpyHostToDevice, s));
                EW_CUDA_CHECK(cudaStreamSynchronize(s));  // host staging goes out of scope
            }
        } else {
            sort_rows_desc(m, fwd.get(), inv.get(), slen.get(), s, nullptr);
        }
    }
    auto out = std::make_shared<CsrData>();
    out->nrows = n;
    out->ncols = m.ncols;
    out->nnz = nnz;
    out->maxrow = m.maxrow;
    out->ro.alloc(n + 1);
    out->ci.alloc(nnz);
    out->v.alloc(nnz);
    EW_CUDA_CHECK(cudaMemcpyAsync(out->ro.get(), m.ro.get(), (n + 1) * sizeof(int64_t),
                                  cudaMemcpyDeviceToDevice, s));
    if (nnz) {
        Scratch<int32_t> tmp(sort_within_rows ? nnz : 0, s);
        int32_t* cdst = sort_within_rows ? tmp.get() : out->ci.get();
        if (renumber) {
            renumber_kernel<<<grid_for(nnz), kBlock, 0, s>>>(m.ci.get(), inv.get(), cdst, nnz);
            launched("renumber_kernel");
        } else {
            EW_CUDA_CHECK(cudaMemcpyAsync(cdst, m.ci.get(), nnz * 4, cudaMemcpyDeviceToDevice, s));
        }
        if (sort_within_rows) {
            row_rank_sort_kernel<<<fill_grid(n), 256, 0, s>>>(m.ro.get(), tmp.get(), m.v.get(), out->ci.get(),
                                                              out->v.get(), dst_of ? dst_of->get() : nullptr, n);
            launched("row_rank_sort_kernel");
        } else {
            EW_CUDA_CHECK(cudaMemcpyAsync(out->v.get(), m.v.get(), nnz * sizeof(double),
                                          cudaMemcpyDeviceToDevice, s));
            if (dst_of) {
                iota_kernel<<<grid_for(nnz), kBlock, 0, s>>>(dst_of->get(), nnz);
                launched("iota_kernel");
            }
        }
    }
    if (fwd_out && renumber && n)
        EW_CUDA_CHECK(cudaMemcpyAsync(fwd_out, fwd.get(), n * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    EW_CUDA_CHECK(cudaStreamSynchronize(s));
    return out;
}

// 16-bit columns for the K1 warps whose real columns lie within 0xFFFF of
// each other (mesh matrices in a natural or banded order: all but a few
// warps of boundary rows); those warps stream 10 instead of 12 bytes per
// slot, the rest keep the int32 slab (col_base < 0). Only for slabs that
// stream from HBM (over 64 MB of values + columns: config 2's SpMV 163.6 ->
// 158.0 us); on L2-resident ones the offset decode sits in the gather's
// dependency chain and costs more than the bytes it saves (config 1: 5.9 ->
// 6.3 us). Skipped when over a quarter of the slots are in wide warps.
// EW_COMPACT=0: off; EW_COMPACT=2: at any size (tests).
static void compact_layout(LayoutData& l, cudaStream_t s) {
    static const int mode = [] {
        const char* e = std::getenv("EW_COMPACT");
        return e ? std::atoi(e) : 1;
    }();
    if (mode == 0 || l.nslots == 0) return;
    if (mode == 1 && l.nslots * 12 <= (64ll << 20)) return;
    DevBuf<int32_t> base(l.nwarps);
    Scratch<int64_t> fail(1, s);  // slots of warps whose columns span >= 0xFFFF
    EW_CUDA_CHECK(cudaMemsetAsync(fail.get(), 0, sizeof(int64_t), s));
    compact_range_kernel<<<fill_grid(l.nwarps), 256, 0, s>>>(l.cols.get(), l.warp_offset.get(), l.maxrows.get(),
                                                             l.rows_in_warp.get(), l.slen.get(), l.ws, l.ws_log2,
                                                             l.nwarps, base.get(), fail.get());
    launched("compact_range_kernel");
    int64_t wide = 0;
    EW_CUDA_CHECK(cudaMemcpyAsync(&wide, fail.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    EW_CUDA_CHECK(cudaStreamSynchronize(s));
    static const double min_narrow = [] {
        const char* e = std::getenv("EW_COMPACT_MIN");  // A/B runs: least narrow share
        return e ? std::atof(e) : 0.75;
    }();
    if (double(l.stored_slots - wide) < min_narrow * double(l.stored_slots)) return;  // mostly wide warps
    l.cols16.alloc(l.nslots);
    compact_encode_kernel<<<fill_grid(l.nwarps), 256, 0, s>>>(l.cols.get(), l.warp_offset.get(), l.maxrows.get(),
                                                              l.rows_in_warp.get(), l.slen.get(), l.ws, l.ws_log2,
                                                              l.nwarps, base.get(), l.cols16.get());
    launched("compact_encode_kernel");
    l.col_base = std::move(base);
    l.narrow_slots = l.stored_slots - wide;  // stored slots of the narrow warps
    l.compact = 1;
}

// ---- grouped columns for K1 -------------------------------------------------
// One thread per sorted row (a hardware warp = a layout warp, ws = 32): a lane
// starts a group unless its column list (all maxrows steps, padding
// included) equals the previous lane's. lane_grp = its group, ngrp per warp.
__global__ void group_lanes_kernel(const int32_t* __restrict__ cols, const int64_t* __restrict__ woff,
                                   const int32_t* __restrict__ maxrows, const int32_t* __restrict__ rows_in_warp,
                                   int64_t nrows, int64_t nwarps, uint8_t* __restrict__ lane_grp,
                                   uint8_t* __restrict__ ngrp, int64_t* __restrict__ gsize) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t w = p >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= nwarps) return;  // whole hardware warps exit together
    const int32_t mx = maxrows[w], riw = rows_in_warp[w];
    const int64_t off = woff[w];
    bool start = lane == 0;
    if (lane > 0 && lane < riw) {
        bool same = true;
        for (int32_t j = 0; j < mx && same; ++j) same = cols[off + int64_t(j) * 32 + lane] == cols[off + int64_t(j) * 32 + lane - 1];
        start = !same;
    }
    const unsigned starts = __ballot_sync(0xffffffffu, start);
    const int g = __popc(starts & (0xffffffffu >> (31 - lane))) - 1;
    if (p < nrows) lane_grp[p] = static_cast<uint8_t>(g);
    if (lane == 0) {
        const int ng = __popc(starts);
        ngrp[w] = static_cast<uint8_t>(ng);
        gsize[w] = int64_t(mx) * ng;
    }
}

// The leader lane of each group copies its column list into the grouped slab
// (16-bit offsets from col_base when `base` is given, 0xFFFF = padding).
__global__ void group_fill_kernel(const int32_t* __restrict__ cols, const int64_t* __restrict__ woff,
                                  const int32_t* __restrict__ maxrows, const int32_t* __restrict__ rows_in_warp,
                                  const int32_t* __restrict__ slen, int64_t nwarps, const uint8_t* __restrict__ lane_grp,
                                  const uint8_t* __restrict__ ngrp, const int64_t* __restrict__ goff,
                                  const int32_t* __restrict__ base, int32_t* __restrict__ g32,
                                  uint16_t* __restrict__ g16) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t w = p >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= nwarps) return;
    const int32_t mx = maxrows[w], riw = rows_in_warp[w];
    const int g = lane < riw ? lane_grp[p] : -1;
    const int prev = __shfl_up_sync(0xffffffffu, g, 1);
    if (lane >= riw || (lane > 0 && prev == g)) return;  // not a group leader
    if (g16 && base[w] < 0) return;  // a wide warp of a compact layout reads its own int32 columns
    const int64_t off = woff[w], go = goff[w];
    const int ng = ngrp[w];
    const int32_t len = slen[p];
    for (int32_t j = 0; j < mx; ++j) {
        const int32_t c = cols[off + int64_t(j) * 32 + lane];
        const int64_t at = go + int64_t(j) * ng + g;
        if (g16) g16[at] = j < len ? static_cast<uint16_t>(c - base[w]) : uint16_t(0xFFFF);
        else g32[at] = c;
    }
}

// Grouped columns for a K1 slab over 64 MB (int32 or compact layouts; a
// compact layout's wide warps keep reading their int32 columns) when lanes
// share enough lists: the slab's
// column bytes drop to ngrp/32 (3-DOF elasticity: 11.3 groups per 32 lanes;
// 12 -> 9.4 B/slot int32, 10 -> 8.7 with 16-bit offsets). EW_GROUPED=0: off.
static void group_layout(LayoutData& l, cudaStream_t s) {
    static const int mode = [] {
        const char* e = std::getenv("EW_GROUPED");
        return e ? std::atoi(e) : 1;
    }();
    if (mode == 0 || l.kind != EW_LAYOUT_K1 || l.row_major || l.ws != 32 || !l.sorted || l.nwarps == 0) return;
    if (mode == 1 && l.nslots * 12 <= (64ll << 20)) return;
    const int64_t nw = l.nwarps;
    DevBuf<uint8_t> lg(l.nrows), ng(nw);
    Scratch<int64_t> gsize(nw, s);
    group_lanes_kernel<<<grid_for(nw * 32), kBlock, 0, s>>>(l.cols.get(), l.warp_offset.get(), l.maxrows.get(),
                                                            l.rows_in_warp.get(), l.nrows, nw, lg.get(), ng.get(),
                                                            gsize.get());
    launched("group_lanes_kernel");
    DevBuf<int64_t> go(nw);
    exclusive_scan_i64(gsize.get(), go.get(), nw, s);
    const int64_t total = read_scalar(go.get() + nw - 1, s) + read_scalar(gsize.get() + nw - 1, s);
    if (double(total) > 0.75 * double(l.nslots)) return;  // too few shared lists to pay
    if (l.compact) l.gcols16.alloc(total);
    else l.gcols.alloc(total);
    group_fill_kernel<<<grid_for(nw * 32), kBlock, 0, s>>>(l.cols.get(), l.warp_offset.get(), l.maxrows.get(),
                                                           l.rows_in_warp.get(), l.slen.get(), nw, lg.get(), ng.get(),
                                                           go.get(), l.compact ? l.col_base.get() : nullptr,
                                                           l.gcols.get(), l.gcols16.get());
    launched("group_fill_kernel");
    int64_t bytes = 4 * total;
    if (l.compact) {  // narrow warps stream 2 B per grouped entry, wide ones their own int32 slab
        std::vector<int64_t> gs(nw), wo(nw);
        std::vector<int32_t> b(nw), mxs(nw);
        EW_CUDA_CHECK(cudaMemcpyAsync(gs.data(), gsize.get(), nw * 8, cudaMemcpyDeviceToHost, s));
        EW_CUDA_CHECK(cudaMemcpyAsync(b.data(), l.col_base.get(), nw * 4, cudaMemcpyDeviceToHost, s));
        EW_CUDA_CHECK(cudaMemcpyAsync(mxs.data(), l.maxrows.get(), nw * 4, cudaMemcpyDeviceToHost, s));
        EW_CUDA_CHECK(cudaStreamSynchronize(s));
        bytes = 0;
        for (int64_t w = 0; w < nw; ++w) bytes += b[w] >= 0 ? 2 * gs[w] : 4 * int64_t(mxs[w]) * l.ws;
    }
    l.lane_grp = std::move(lg);
    l.ngrp = std::move(ng);
    l.goff = std::move(go);
    l.grouped_slots = total;
    l.grouped_col_bytes = bytes;
    l.grouped = 1;
}

int32_t head_mx() {
    static const int32_t v = [] {
        const char* e = std::getenv("EW_K1_HEAD");  // 0: off; else the head's row-length bound
        return e ? std::max(0, std::atoi(e)) : 64;
    }();
    return v;
}

// ---- the int32 column slab of compact / grouped layouts ---------------------
struct ColForms {
    const int64_t* woff;
    const int32_t* maxrows;
    const int32_t* rows_in_warp;
    const int32_t* cols;       // full slab, or the wide warps' slabs (col_shift)
    const int64_t* col_shift;  // nullptr: cols is the full slab (or empty)
    const uint16_t* cols16;
    const int32_t* col_base;   // compact
    const uint8_t* lane_grp;   // grouped
    const uint8_t* ngrp;
    const int64_t* goff;
    const int32_t* gcols;
    const uint16_t* gcols16;
    int32_t ws, ws_log2;
    int64_t nwarps;
    int compact, grouped, full;
};

// The int32 column of each stored slot from the form the kernels read (one
// hardware warp per layout warp, lanes striding its slots): the wide warps'
// own slab, the 16-bit offsets (0xFFFF = padding = column 0), or the grouped
// lists; lanes past the warp's rows are padding (column 0) as in fill_kernel.
__global__ void decode_cols_kernel(ColForms f, int32_t* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nhw = (gridDim.x * (int64_t)blockDim.x) >> 5;
    for (int64_t w = gw; w < f.nwarps; w += nhw) {
        const int64_t n = int64_t(f.maxrows[w]) * f.ws, off = f.woff[w];
        const int32_t nr = f.rows_in_warp[w];
        const int32_t b = f.compact ? f.col_base[w] : 0;
        for (int64_t i = lane; i < n; i += 32) {
            const int32_t l = static_cast<int32_t>(i & (f.ws - 1));
            const int64_t j = i >> f.ws_log2;
            int32_t c;
            if (f.full) {
                c = f.cols[off + i];
            } else if (f.compact && b < 0) {
                c = f.cols[f.col_shift[w] + off + i];
            } else if (l >= nr) {
                c = 0;
            } else if (f.grouped) {
                const int64_t g = f.goff[w] + j * f.ngrp[w] + f.lane_grp[w * f.ws + l];
                if (f.compact) {
                    const uint16_t d = f.gcols16[g];
                    c = d == 0xFFFFu ? 0 : b + static_cast<int32_t>(d);
                } else {
                    c = f.gcols[g];
                }
            } else {
                const uint16_t d = f.cols16[off + i];
                c = d == 0xFFFFu ? 0 : b + static_cast<int32_t>(d);
            }
            out[off + i] = c;
        }
    }
}

// Copies each wide warp's int32 slab to its place in the reduced slab.
__global__ void wide_copy_kernel(const int32_t* __restrict__ cols, const int64_t* __restrict__ woff,
                                 const int32_t* __restrict__ maxrows, const int32_t* __restrict__ base,
                                 const int64_t* __restrict__ shift, int32_t ws, int64_t nwarps,
                                 int32_t* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nhw = (gridDim.x * (int64_t)blockDim.x) >> 5;
    for (int64_t w = gw; w < nwarps; w += nhw) {
        if (base[w] >= 0) continue;
        const int64_t n = int64_t(maxrows[w]) * ws, off = woff[w];
        for (int64_t i = lane; i < n; i += 32) out[shift[w] + off + i] = cols[off + i];
    }
}

__global__ void wide_size_kernel(const int32_t* __restrict__ maxrows, const int32_t* __restrict__ base,
                                 int32_t ws, int64_t nwarps, int64_t* __restrict__ size) {
    const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (w < nwarps) size[w] = base[w] < 0 ? int64_t(maxrows[w]) * ws : 0;
}

__global__ void shift_kernel(const int64_t* __restrict__ woff, int64_t nwarps, int64_t* __restrict__ shift) {
    const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (w < nwarps) shift[w] -= woff[w];  // wide offset - slab offset
}

void decode_columns(const LayoutData& l, int32_t* out, cudaStream_t s) {
    if (l.nslots == 0) return;
    EW_CUDA_CHECK(cudaMemsetAsync(out, 0, l.nslots * sizeof(int32_t), s));  // alignment gaps
    ColForms f{l.warp_offset.get(), l.maxrows.get(), l.rows_in_warp.get(), l.cols.get(), l.col_shift.get(),
               l.cols16.get(), l.col_base.get(), l.lane_grp.get(), l.ngrp.get(), l.goff.get(), l.gcols.get(),
               l.gcols16.get(), l.ws, l.ws_log2, l.nwarps, l.compact, l.grouped, l.cols_full ? 1 : 0};
    if (l.nwarps) {
        decode_cols_kernel<<<fill_grid(l.nwarps), 256, 0, s>>>(f, out);
        launched("decode_cols_kernel");
    }
}

void restore_columns(LayoutData& l, cudaStream_t s) {
    if (l.cols_full) return;
    DevBuf<int32_t> full(l.nslots);
    decode_columns(l, full.get(), s);
    EW_CUDA_CHECK(cudaStreamSynchronize(s));
    l.cols = std::move(full);
    l.col_shift.release();
    l.cols_full = true;
}

// Drops the column slabs the kernels of a compact or grouped layout no
// longer read: a compact layout keeps int32 columns for its wide warps only
// (and, grouped, no per-slot 16-bit offsets either: config 2 14.7 -> ~8.8
// bytes per slot), a grouped int32 one no int32 slab (config 5 whole: 18 GB),
// unless the SpMV form chosen for it (the cooperative K1) streams the int32
// slab. Export, the host-buffer pipeline's
// plan and the split-x K1 decode or restore it (decode_columns).
static void shrink_columns(LayoutData& l, cudaStream_t s) {
    static const bool keep = [] {
        const char* e = std::getenv("EW_KEEP_INT32_COLS");  // A/B runs
        return e && e[0] == '1';
    }();
    if (keep || !l.cols_full || !(l.compact || l.grouped) || l.nwarps == 0 || spmv_reads_int32(l)) return;
    if (!l.compact) {  // grouped int32: the kernels read gcols
        l.cols.release();
        l.cols_full = false;
        return;
    }
    const int64_t nw = l.nwarps;
    Scratch<int64_t> size(nw, s);
    wide_size_kernel<<<grid_for(nw), kBlock, 0, s>>>(l.maxrows.get(), l.col_base.get(), l.ws, nw, size.get());
    launched("wide_size_kernel");
    DevBuf<int64_t> shift(nw);
    exclusive_scan_i64(size.get(), shift.get(), nw, s);
    const int64_t total = read_scalar(shift.get() + nw - 1, s) + read_scalar(size.get() + nw - 1, s);
    shift_kernel<<<grid_for(nw), kBlock, 0, s>>>(l.warp_offset.get(), nw, shift.get());
    launched("shift_kernel");
    DevBuf<int32_t> wide(total);
    if (total) {
        wide_copy_kernel<<<fill_grid(nw), 256, 0, s>>>(l.cols.get(), l.warp_offset.get(), l.maxrows.get(),
                                                         l.col_base.get(), shift.get(), l.ws, nw, wide.get());
        launched("wide_copy_kernel");
    }
    EW_CUDA_CHECK(cudaStreamSynchronize(s));
    l.cols = std::move(wide);
    l.col_shift = std::move(shift);
    l.cols_full = false;
    if (l.grouped) l.cols16.release();  // the grouped lists replace the per-slot offsets too
}

std::shared_ptr<LayoutData> build_layout(const CsrData& m, int kind, const ew_warp_config& cfg,
                                         int64_t threshold, bool sort_rows, bool row_major,
                                         cudaStream_t s) {
    validate_config(cfg);
    require(kind == EW_LAYOUT_K1 || kind == EW_LAYOUT_K2, "layout kind must be k1 or k2");
    if (kind == EW_LAYOUT_K2) require(threshold >= 1, "build_k2: threshold must be >= 1");
    if (cfg.warp_size > 1024) throw Error(EW_UNSUPPORTED, "warp_size above 1024 has no device mapping");
    auto L = std::make_shared<LayoutData>();
    LayoutData& l = *L;
    const int64_t n = m.nrows;
    l.kind = kind;
    l.ws = cfg.warp_size;
    l.ws_log2 = log2_exact(cfg.warp_size);
    l.row_major = (kind == EW_LAYOUT_K1 && row_major) ? 1 : 0;
    l.sorted = sort_rows ? 1 : 0;
    l.segment_bytes = cfg.segment_bytes;
    l.align = cfg.align_warp_offsets ? 1 : 0;
    l.nrows = n;
    l.ncols = m.ncols;
    l.nnz = m.nnz;
    l.threshold = kind == EW_LAYOUT_K2 ? threshold : 0;
    l.fwd.alloc(n);
    l.inv.alloc(n);
    l.slen.alloc(n);
    const int64_t unit = l.align ? std::max<int64_t>(1, cfg.segment_bytes / 4) : 1;

    Scratch<unsigned long long> counters(2, s);  // n_active, stored_slots
    Scratch<int> max_red(1, s);
    EW_CUDA_CHECK(cudaMemsetAsync(counters.get(), 0, 2 * sizeof(unsigned long long), s));
    EW_CUDA_CHECK(cudaMemsetAsync(max_red.get(), 0, sizeof(int), s));
    if (n) {
        if (sort_rows) {
            sort_rows_desc(m, l.fwd.get(), l.inv.get(), l.slen.get(), s, counters.get());
        } else {
            identity_perm_kernel<<<grid_for(n), kBlock, 0, s>>>(m.ro.get(), l.fwd.get(), l.inv.get(),
                                                                l.slen.get(), n, counters.get());
            launched("identity_perm_kernel");
        }
    }

    Scratch<int64_t>* sizes = nullptr;
    std::unique_ptr<Scratch<int64_t>> sizes_owner;
    if (kind == EW_LAYOUT_K1) {
        const int64_t nw = (n + l.ws - 1) / l.ws;
        l.nwarps = nw;
        l.maxrows.alloc(nw);
        l.rows_in_warp.alloc(nw);
        sizes_owner = std::make_unique<Scratch<int64_t>>(nw, s);
        sizes = sizes_owner.get();
        if (nw) {
            k1_meta_kernel<<<grid_for(nw), kBlock, 0, s>>>(l.slen.get(), n, l.ws, nw, unit,
                                                           l.maxrows.get(), l.rows_in_warp.get(),
                                                           sizes->get(), counters.get() + 1);
            launched("k1_meta_kernel");
        }
        l.max_reduction = 1;
    } else {
        int64_t nw = 0;
        if (n) {
            Scratch<int32_t> lanes(n, s), flag(n, s), wid(n, s);
            Scratch<int64_t> run_mark(n, s), run_start(n, s);
            k2_lanes_kernel<<<grid_for(n), kBlock, 0, s>>>(l.slen.get(), n, threshold, l.ws,
                                                           lanes.get(), run_mark.get());
            launched("k2_lanes_kernel");
            size_t bytes = 0;
            EW_CUDA_CHECK(cub::DeviceScan::InclusiveScan(nullptr, bytes, run_mark.get(), run_start.get(),
                                                         cub::Max(), n, s));
            {
                Scratch<unsigned char> tmp(bytes, s);
                EW_CUDA_CHECK(cub::DeviceScan::InclusiveScan(tmp.get(), bytes, run_mark.get(),
                                                             run_start.get(), cub::Max(), n, s));
                launched("cub::DeviceScan::InclusiveScan(max)");
            }
            k2_warp_start_kernel<<<grid_for(n), kBlock, 0, s>>>(lanes.get(), run_start.get(), n, l.ws,
                                                                flag.get());
            launched("k2_warp_start_kernel");
            bytes = 0;
            EW_CUDA_CHECK(cub::DeviceScan::InclusiveSum(nullptr, bytes, flag.get(), wid.get(), n, s));
            {
                Scratch<unsigned char> tmp(bytes, s);
                EW_CUDA_CHECK(cub::DeviceScan::InclusiveSum(tmp.get(), bytes, flag.get(), wid.get(), n, s));
                launched("cub::DeviceScan::InclusiveSum");
            }
            nw = read_scalar(wid.get() + n - 1, s);
            l.nwarps = nw;
            l.rows_offset_warp.alloc(nw);
            l.reduction.alloc(nw);
            l.rows_in_warp.alloc(nw);
            l.maxrows.alloc(nw);
            k2_meta_kernel<<<grid_for(n), kBlock, 0, s>>>(flag.get(), wid.get(), lanes.get(), n,
                                                          l.rows_offset_warp.get(), l.reduction.get());
            launched("k2_meta_kernel");
            sizes_owner = std::make_unique<Scratch<int64_t>>(nw, s);
            sizes = sizes_owner.get();
            k2_meta2_kernel<<<grid_for(nw), kBlock, 0, s>>>(
                l.slen.get(), l.rows_offset_warp.get(), l.reduction.get(), n, nw, l.ws, unit,
                l.rows_in_warp.get(), l.maxrows.get(), sizes->get(), counters.get() + 1, max_red.get());
            launched("k2_meta2_kernel");
            EW_CUDA_CHECK(cudaStreamSynchronize(s));  // scratch freed before the fill allocations
        }
        l.nwarps = nw;
    }

    const int64_t nw = l.nwarps;
    l.warp_offset.alloc(nw);
    if (nw) {
        exclusive_scan_i64(sizes->get(), l.warp_offset.get(), nw, s);
        const int64_t last_off = read_scalar(l.warp_offset.get() + nw - 1, s);
        const int32_t last_mx = read_scalar(l.maxrows.get() + nw - 1, s);
        l.nslots = last_off + int64_t(last_mx) * l.ws;
        // sorted longest-first: warp 0 holds the longest row
        if (kind == EW_LAYOUT_K1 && l.sorted) l.max_mx = read_scalar(l.maxrows.get(), s);
        // a few very long rows: the warps over head_mx() entries (a prefix,
        // maxrows falls with the warp index) go to the cooperative K1
        const int32_t hm = head_mx();
        if (kind == EW_LAYOUT_K1 && l.sorted && !row_major && l.ws == 32 && hm > 0 && l.max_mx > 4 * hm) {
            int64_t lo = 0, hi = nw;  // first warp with maxrows <= hm
            while (lo < hi) {
                const int64_t mid = (lo + hi) / 2;
                if (read_scalar(l.maxrows.get() + mid, s) > hm) lo = mid + 1;
                else hi = mid;
            }
            // at most four 1024-thread CTAs per SM of head: the long-row
            // kernel spends a whole CTA on each layout warp, which pays for
            // the few longest rows, not for a fat band of moderately long
            // ones (the plain K1 keeps those; any split point is valid)
            l.head_warps = std::min<int64_t>(lo, 148 * 4);
            if (lo > 0) {
                l.side = std::make_shared<SideStream>();
                k1_long_setup();
            }
        }
    }
    sizes_owner.reset();
    unsigned long long hc[2];
    int hr = 0;
    EW_CUDA_CHECK(cudaMemcpyAsync(hc, counters.get(), sizeof(hc), cudaMemcpyDeviceToHost, s));
    EW_CUDA_CHECK(cudaMemcpyAsync(&hr, max_red.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    EW_CUDA_CHECK(cudaStreamSynchronize(s));
    l.stored_slots = static_cast<int64_t>(hc[1]);
    if (kind == EW_LAYOUT_K2) l.max_reduction = std::max(1, hr);
    // rows with >= 1 entry; when sorted they are the prefix [0, n_active)
    l.n_active = static_cast<int64_t>(hc[0]);

    l.values.alloc(l.nslots);
    l.cols.alloc(l.nslots);
    if (nw) {
        fill_kernel<<<fill_grid(nw), 256, 0, s>>>(mapper_of(l, m), m.v.get(), m.ci.get(), l.values.get(),
                                                  l.cols.get());
        launched("fill_kernel");
    }
    if (kind == EW_LAYOUT_K1 && !l.row_major && nw) {
        compact_layout(l, s);
        group_layout(l, s);
        shrink_columns(l, s);
    }
    EW_CUDA_CHECK(cudaStreamSynchronize(s));
    return L;
}

void layout_build_slot_map(LayoutData& l, const CsrData& m, cudaStream_t s) {
    require(m.nrows == l.nrows && m.nnz == l.nnz, "value_slot_map: matrix does not match the layout");
    if (l.slot_map.size() == size_t(m.nnz) && m.nnz) return;
    l.slot_map.alloc(m.nnz);
    if (l.nwarps && m.nnz) {
        slot_map_kernel<<<fill_grid(l.nwarps), 256, 0, s>>>(mapper_of(l, m), l.slot_map.get());
        launched("slot_map_kernel");
    }
}

namespace {
void ensure_src_map(LayoutData& l, const CsrData& m, const int64_t* dst_of, cudaStream_t s) {
    require(m.nrows == l.nrows && m.nnz == l.nnz, "refresh: matrix does not match the layout");
    if (l.src_map.size() == size_t(l.nslots)) return;
    // the r / rs operand keeps m's row offsets, so m maps the operand's
    // entries to slots; orig_of = dst_of^-1 takes them back to m's entries
    Scratch<int64_t> orig_of(dst_of ? m.nnz : 0, s);
    if (dst_of && m.nnz) {
        invert_kernel<<<grid_for(m.nnz), kBlock, 0, s>>>(dst_of, orig_of.get(), m.nnz);
        launched("invert_kernel");
    }
    l.src_map.alloc(l.nslots);
    if (l.nwarps) {
        src_map_kernel<<<fill_grid(l.nwarps), 256, 0, s>>>(mapper_of(l, m), dst_of ? orig_of.get() : nullptr,
                                                           l.src_map.get());
        launched("src_map_kernel");
    }
    EW_CUDA_CHECK(cudaStreamSynchronize(s));  // orig_of is freed on return
}
}  // namespace

void layout_src_map(const LayoutData& l, const CsrData& m, const int64_t* orig_of, int64_t* out, cudaStream_t s) {
    if (!l.nwarps) return;
    src_map_kernel<<<fill_grid(l.nwarps), 256, 0, s>>>(mapper_of(l, m), orig_of, out);
    launched("src_map_kernel");
}

void layout_refresh_values_reordered(LayoutData& l, const CsrData& m, const int64_t* dst_of, cudaStream_t s) {
    ensure_src_map(l, m, dst_of, s);
    if (!l.nslots) return;
    refresh_gather_kernel<<<grid_for(l.nslots), kBlock, 0, s>>>(l.src_map.get(), m.v.get(), l.values.get(),
                                                                l.nslots);
    launched("refresh_gather_kernel");
}

void layout_refresh_values(LayoutData& l, const CsrData& m, cudaStream_t s) {
    layout_refresh_values_reordered(l, m, nullptr, s);
}

std::shared_ptr<LayoutData> import_layout(const ew_layout_desc& d, cudaStream_t s) {
    require(d.kind == EW_LAYOUT_K1 || d.kind == EW_LAYOUT_K2, "layout kind must be k1 or k2");
    require(d.warp_size > 0 && (d.warp_size & (d.warp_size - 1)) == 0, "warp_size must be a power of two");
    if (d.warp_size > 1024) throw Error(EW_UNSUPPORTED, "warp_size above 1024 has no device mapping");
    require(d.nrows >= 0 && d.ncols >= 0 && d.nwarps >= 0 && d.nslots >= 0, "negative layout sizes");
    if (d.nrows > 0x7fffffff || d.ncols > 0x7fffffff)
        throw Error(EW_UNSUPPORTED, "device path supports at most 2^31-1 rows and columns");
    auto L = std::make_shared<LayoutData>();
    LayoutData& l = *L;
    l.kind = d.kind;
    l.ws = d.warp_size;
    l.ws_log2 = log2_exact(d.warp_size);
    l.row_major = d.kind == EW_LAYOUT_K1 && d.row_major ? 1 : 0;
    l.nrows = d.nrows;
    l.ncols = d.ncols;
    l.nnz = d.nnz;
    l.nwarps = d.nwarps;
    l.nslots = d.nslots;
    l.threshold = d.threshold;
    const int64_t n = d.nrows, nw = d.nwarps, ns = d.nslots;
    auto narrow = [](const int64_t* src, int64_t k, const char* what, int64_t lo, int64_t hi) {
        std::vector<int32_t> out(static_cast<size_t>(k));
        for (int64_t i = 0; i < k; ++i) {
            require(src[i] >= lo && src[i] <= hi, std::string("layout ") + what + " out of range");
            out[i] = static_cast<int32_t>(src[i]);
        }
        return out;
    };
    auto up32 = [&](DevBuf<int32_t>& dst, const std::vector<int32_t>& h) {
        dst.alloc(h.size());
        if (!h.empty())
            EW_CUDA_CHECK(cudaMemcpyAsync(dst.get(), h.data(), h.size() * 4, cudaMemcpyHostToDevice, s));
    };
    require(d.forward && d.sorted_row_length && d.warp_offset && d.maxrows && d.rows_in_warp,
            "layout arrays missing");
    require(ns == 0 || (d.values && d.col_indices), "layout arrays missing");
    const auto h_fwd = narrow(d.forward, n, "row_perm", 0, n - 1);
    const auto h_slen = narrow(d.sorted_row_length, n, "sorted_row_length", 0, 0x7fffffff);
    const auto h_mx = narrow(d.maxrows, nw, "maxrows", 0, 0x7fffffff);
    const auto h_riw = narrow(d.rows_in_warp, nw, "rows_in_warp", 0, l.ws);
    const auto h_cols = narrow(d.col_indices, ns, "col_indices", 0, std::max<int64_t>(0, d.ncols - 1));
    std::vector<int32_t> h_inv(static_cast<size_t>(n), -1);
    for (int64_t p = 0; p < n; ++p) {
        require(h_inv[h_fwd[p]] == -1, "permutation not a bijection");
        h_inv[h_fwd[p]] = static_cast<int32_t>(p);
    }
    // every slot the kernel touches must be inside the arrays
    int64_t stored = 0;
    int32_t max_red = 1;
    std::vector<int32_t> h_red, h_row;
    if (d.kind == EW_LAYOUT_K2) {
        require(d.reduction && d.rows_offset_warp, "k2 layout needs reduction and rows_offset_warp");
        h_red = narrow(d.reduction, nw, "reduction", 1, l.ws);
        h_row = narrow(d.rows_offset_warp, nw, "rows_offset_warp", 0, std::max<int64_t>(0, n));
    }
    for (int64_t w = 0; w < nw; ++w) {
        const int32_t red = d.kind == EW_LAYOUT_K2 ? h_red[w] : 1;
        require((red & (red - 1)) == 0, "reduction must be a power of two");
        max_red = std::max(max_red, red);
        require(d.warp_offset[w] >= 0 && d.warp_offset[w] + int64_t(h_mx[w]) * l.ws <= ns,
                "warp slab outside the value array");
        const int64_t first = d.kind == EW_LAYOUT_K2 ? h_row[w] : w * l.ws;
        require(first + h_riw[w] <= n, "warp rows outside the matrix");
        require(int64_t(h_riw[w]) * red <= l.ws, "warp rows exceed the warp size");
        stored += int64_t(h_mx[w]) * red * h_riw[w];
    }
    if (d.kind == EW_LAYOUT_K1) {
        // K1 grouping is positional (warp_layout.cpp:47-52); the device
        // kernel maps thread p to warp p / ws, so the import must match it
        require(nw == (n + l.ws - 1) / l.ws, "k1 layout must have ceil(nrows / warp_size) warps");
        for (int64_t w = 0; w < nw; ++w)
            require(h_riw[w] == std::min<int64_t>(l.ws, n - w * l.ws), "k1 rows_in_warp mismatch");
    }
    l.imported = true;
    l.stored_slots = stored;
    l.max_reduction = max_red;
    bool sorted = true;
    int64_t active = 0;
    for (int64_t p = 0; p < n; ++p) {
        if (p && h_slen[p] > h_slen[p - 1]) sorted = false;
        if (h_slen[p] > 0) ++active;
    }
    l.sorted = sorted ? 1 : 0;
    l.n_active = active;
    up32(l.fwd, h_fwd);
    up32(l.inv, h_inv);
    up32(l.slen, h_slen);
    up32(l.maxrows, h_mx);
    up32(l.rows_in_warp, h_riw);
    up32(l.cols, h_cols);
    if (d.kind == EW_LAYOUT_K2) {
        up32(l.reduction, h_red);
        up32(l.rows_offset_warp, h_row);
    }
    l.warp_offset.alloc(nw);
    if (nw) EW_CUDA_CHECK(cudaMemcpyAsync(l.warp_offset.get(), d.warp_offset, nw * 8, cudaMemcpyHostToDevice, s));
    l.values.alloc(ns);
    if (ns) EW_CUDA_CHECK(cudaMemcpyAsync(l.values.get(), d.values, ns * 8, cudaMemcpyHostToDevice, s));
    EW_CUDA_CHECK(cudaStreamSynchronize(s));
    return L;
}

const void* kernel_anchor_layout() { return reinterpret_cast<const void*>(&sort_keys_kernel); }

}  // namespace ew

// Locality row order for the reordered (r / rs) kernels: a level-synchronous
// Cuthill-McKee BFS on the device, then the reference's stable longest-first
// sort applied on top of it (permutation.cpp:49-55 with the BFS order as the
// tie-break instead of the row id).
//
// Why: on B200 the K1 SpMV of a randomly numbered mesh (config 4) is bound by
// L2 sector throughput, not HBM -- every x gather of a warp touches its own
// 32-byte sector. Grouping mesh neighbours into the same layout warp (and
// storing the vectors in that order) turns those gathers into L1 hits. Each
// row keeps the reference's entry order (original for r, ascending sorted
// index for rs, reorder.cpp:8-43), so every row sum is the reference's, bit
// for bit; only which rows share a warp -- and therefore padding -- changes.
//
// The order is deterministic: a frontier node's unvisited neighbours take the
// smallest parent position (atomicMin), each level is sorted by (parent
// position, row id), disconnected parts restart at their lowest row id.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "ew_internal.cuh"

namespace ew {

namespace {

constexpr uint32_t kUnseen = 0xffffffffu;
constexpr int kMaxRestarts = 64;  // then the rest is appended in row order

__global__ void start_kernel(const int64_t* __restrict__ ro, const int32_t* __restrict__ seen, int64_t n,
                             unsigned long long* best) {
    // lowest degree first (a mesh corner), then lowest row id; one atomic per warp
    unsigned long long key = ~0ull;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        if (seen[r]) continue;
        const int64_t len = ro[r + 1] - ro[r];
        const unsigned long long k =
            (static_cast<unsigned long long>(len < 0xffffffffLL ? len : 0xffffffffLL) << 32) |
            static_cast<unsigned long long>(r);
        key = k < key ? k : key;
    }
    for (int o = 16; o; o >>= 1) {
        const unsigned long long other = __shfl_down_sync(0xffffffffu, key, o);
        key = other < key ? other : key;
    }
    if ((threadIdx.x & 31) == 0 && key != ~0ull) atomicMin(best, key);
}

__global__ void seed_kernel(const unsigned long long* best, int32_t* order, int64_t at, int32_t* seen) {
    const int32_t r = static_cast<int32_t>(*best & 0xffffffffull);
    order[at] = r;
    seen[r] = 1;
}

// One warp per frontier node: each unvisited neighbour records the smallest
// parent position; the first discoverer appends it to `next`.
__global__ void expand_kernel(const int64_t* __restrict__ ro, const int32_t* __restrict__ ci,
                              const int32_t* __restrict__ order, int64_t head, int64_t tail, int64_t n,
                              const int32_t* __restrict__ seen, uint32_t* __restrict__ parent,
                              int32_t* __restrict__ next, unsigned long long* count) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nhw = (gridDim.x * (int64_t)blockDim.x) >> 5;
    for (int64_t pos = head + gw; pos < tail; pos += nhw) {
        const int32_t r = order[pos];
        for (int64_t k = ro[r] + lane; k < ro[r + 1]; k += 32) {
            const int32_t u = ci[k];
            if (u >= n || seen[u]) continue;
            const uint32_t old = atomicMin(parent + u, static_cast<uint32_t>(pos));
            if (old == kUnseen) next[atomicAdd(count, 1ull)] = u;
        }
    }
}

__global__ void level_keys_kernel(const int32_t* __restrict__ next, const uint32_t* __restrict__ parent,
                                  uint64_t* __restrict__ keys, int64_t cnt) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= cnt) return;
    const int32_t u = next[i];
    keys[i] = (static_cast<uint64_t>(parent[u]) << 32) | static_cast<uint32_t>(u);
}

__global__ void level_append_kernel(const uint64_t* __restrict__ keys, int32_t* __restrict__ order, int64_t at,
                                    int32_t* __restrict__ seen, int64_t cnt) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= cnt) return;
    const int32_t u = static_cast<int32_t>(keys[i] & 0xffffffffull);
    order[at + i] = u;
    seen[u] = 1;
}

__global__ void unseen_flags_kernel(const int32_t* __restrict__ seen, int64_t* __restrict__ flag, int64_t n) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r < n) flag[r] = seen[r] ? 0 : 1;
}

__global__ void append_unseen_kernel(const int32_t* __restrict__ seen, const int64_t* __restrict__ at,
                                     int32_t* __restrict__ order, int64_t base, int64_t n) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r < n && !seen[r]) order[base + at[r]] = static_cast<int32_t>(r);
}

// stable longest-first sort keyed on the locality order
__global__ void order_keys_kernel(const int64_t* __restrict__ ro, const int32_t* __restrict__ order,
                                  uint32_t* __restrict__ keys, int64_t n, int32_t maxrow) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int32_t r = order[k];
    keys[k] = static_cast<uint32_t>(maxrow - static_cast<int32_t>(ro[r + 1] - ro[r]));
}

__global__ void invert_perm_kernel(const int32_t* __restrict__ fwd, int32_t* __restrict__ inv,
                                   int64_t* __restrict__ len, const int64_t* __restrict__ ro, int64_t n) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int32_t r = fwd[k];
    inv[r] = static_cast<int32_t>(k);
    len[k] = ro[r + 1] - ro[r];
}

__global__ void compose_kernel(const int32_t* __restrict__ a, const int32_t* __restrict__ b,
                               int32_t* __restrict__ out, int64_t n) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n) out[k] = a[b[k]];  // out = a o b
}

// Row k of the output is row fwd[k] of `in`, entries in their order, columns
// mapped through cmap. One warp per output row.
__global__ void permute_rows_kernel(const int64_t* __restrict__ ro, const int32_t* __restrict__ ci,
                                    const double* __restrict__ v, const int32_t* __restrict__ fwd,
                                    const int32_t* __restrict__ cmap, const int64_t* __restrict__ ro_out,
                                    int32_t* __restrict__ ci_out, double* __restrict__ v_out, int64_t n) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nhw = (gridDim.x * (int64_t)blockDim.x) >> 5;
    for (int64_t k = gw; k < n; k += nhw) {
        const int32_t r = fwd[k];
        const int64_t lo = ro[r], len = ro[r + 1] - lo, dst = ro_out[k];
        for (int64_t j = lane; j < len; j += 32) {
            ci_out[dst + j] = cmap[ci[lo + j]];
            v_out[dst + j] = v[lo + j];
        }
    }
}

unsigned warp_grid(int64_t nwarps) {
    int64_t g = (nwarps + 7) / 8;
    if (g > 148 * 32) g = 148 * 32;
    return static_cast<unsigned>(g < 1 ? 1 : g);
}

template <typename T>
T to_host(const T* d, cudaStream_t s) {
    T h{};
    EW_CUDA_CHECK(cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, s));
    EW_CUDA_CHECK(cudaStreamSynchronize(s));
    return h;
}

}  // namespace

void locality_order(const CsrData& m, int32_t* order, cudaStream_t s) {
    const int64_t n = m.nrows;
    require(m.nrows == m.ncols, "locality order: matrix must be square");
    if (n == 0) return;
    Scratch<int32_t> seen(n, s), next(n, s);
    Scratch<uint32_t> parent(n, s);
    Scratch<unsigned long long> counters(2, s);  // [0] level size, [1] start key
    EW_CUDA_CHECK(cudaMemsetAsync(seen.get(), 0, n * sizeof(int32_t), s));
    EW_CUDA_CHECK(cudaMemsetAsync(parent.get(), 0xff, n * sizeof(uint32_t), s));
    int end_bit = 32;
    while (end_bit < 64 && (int64_t{1} << (end_bit - 32)) < n) ++end_bit;  // parent bits above the id

    int64_t tail = 0;
    int restarts = 0;
    while (tail < n && restarts < kMaxRestarts) {
        EW_CUDA_CHECK(cudaMemsetAsync(counters.get() + 1, 0xff, sizeof(unsigned long long), s));
        start_kernel<<<std::min<unsigned>(grid_for(n), 148 * 8), kBlock, 0, s>>>(m.ro.get(), seen.get(), n, counters.get() + 1);
        launched("start_kernel");
        seed_kernel<<<1, 1, 0, s>>>(counters.get() + 1, order, tail, seen.get());
        launched("seed_kernel");
        ++restarts;
        int64_t head = tail++;
        while (head < tail) {
            EW_CUDA_CHECK(cudaMemsetAsync(counters.get(), 0, sizeof(unsigned long long), s));
            expand_kernel<<<warp_grid(tail - head), 256, 0, s>>>(m.ro.get(), m.ci.get(), order, head, tail, n,
                                                                 seen.get(), parent.get(), next.get(),
                                                                 counters.get());
            launched("expand_kernel");
            const int64_t cnt = static_cast<int64_t>(to_host(counters.get(), s));
            head = tail;
            if (cnt == 0) break;
            Scratch<uint64_t> keys(cnt, s), sorted(cnt, s);
            level_keys_kernel<<<grid_for(cnt), kBlock, 0, s>>>(next.get(), parent.get(), keys.get(), cnt);
            launched("level_keys_kernel");
            size_t bytes = 0;
            EW_CUDA_CHECK(cub::DeviceRadixSort::SortKeys(nullptr, bytes, keys.get(), sorted.get(), cnt, 0, end_bit, s));
            Scratch<unsigned char> tmp(bytes, s);
            EW_CUDA_CHECK(
                cub::DeviceRadixSort::SortKeys(tmp.get(), bytes, keys.get(), sorted.get(), cnt, 0, end_bit, s));
            launched("cub::DeviceRadixSort::SortKeys");
            level_append_kernel<<<grid_for(cnt), kBlock, 0, s>>>(sorted.get(), order, tail, seen.get(), cnt);
            launched("level_append_kernel");
            tail += cnt;
        }
    }
    if (tail < n) {  // many small components: the rest in row order
        Scratch<int64_t> flag(n, s), at(n, s);
        unseen_flags_kernel<<<grid_for(n), kBlock, 0, s>>>(seen.get(), flag.get(), n);
        launched("unseen_flags_kernel");
        size_t bytes = 0;
        EW_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, flag.get(), at.get(), n, s));
        Scratch<unsigned char> tmp(bytes, s);
        EW_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, flag.get(), at.get(), n, s));
        launched("cub::DeviceScan::ExclusiveSum");
        append_unseen_kernel<<<grid_for(n), kBlock, 0, s>>>(seen.get(), at.get(), order, tail, n);
        launched("append_unseen_kernel");
    }
    EW_CUDA_CHECK(cudaStreamSynchronize(s));
}

std::shared_ptr<CsrData> locality_operand(const CsrData& m, const CsrData& op, const int32_t* pf, int32_t* qf,
                                          int32_t* qi, cudaStream_t s) {
    const int64_t n = m.nrows, nnz = m.nnz;
    auto out = std::make_shared<CsrData>();
    out->nrows = n;
    out->ncols = n;
    out->nnz = nnz;
    out->maxrow = m.maxrow;
    out->ro.alloc(n + 1);
    out->ci.alloc(nnz);
    out->v.alloc(nnz);
    if (n == 0) {
        EW_CUDA_CHECK(cudaMemsetAsync(out->ro.get(), 0, sizeof(int64_t), s));
        EW_CUDA_CHECK(cudaStreamSynchronize(s));
        return out;
    }
    {  // Q = stable longest-first sort of the locality order
        Scratch<int32_t> lorder(n, s);
        locality_order(m, lorder.get(), s);
        Scratch<uint32_t> keys(n, s), keys_out(n, s);
        order_keys_kernel<<<grid_for(n), kBlock, 0, s>>>(m.ro.get(), lorder.get(), keys.get(), n, m.maxrow);
        launched("order_keys_kernel");
        const int end_bit = std::max(1, log2_exact(int64_t(m.maxrow) + 1));
        size_t bytes = 0;
        EW_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.get(), keys_out.get(), lorder.get(), qf,
                                                      n, 0, end_bit, s));
        Scratch<unsigned char> tmp(bytes, s);
        EW_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, keys.get(), keys_out.get(), lorder.get(),
                                                      qf, n, 0, end_bit, s));
        launched("cub::DeviceRadixSort::SortPairs");
    }
    Scratch<int64_t> len(n, s);
    invert_perm_kernel<<<grid_for(n), kBlock, 0, s>>>(qf, qi, len.get(), m.ro.get(), n);
    launched("invert_perm_kernel");
    {
        size_t bytes = 0;
        EW_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, len.get(), out->ro.get(), n, s));
        Scratch<unsigned char> tmp(bytes, s);
        EW_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, len.get(), out->ro.get(), n, s));
        launched("cub::DeviceScan::ExclusiveSum");
    }
    EW_CUDA_CHECK(cudaMemcpyAsync(out->ro.get() + n, &out->nnz, sizeof(int64_t), cudaMemcpyHostToDevice, s));
    // op's columns are in P numbering (P = sort_rows_desc): P-column c is
    // original column pf[c], which sits at qi[pf[c]] in Q numbering
    Scratch<int32_t> cmap(n, s);
    compose_kernel<<<grid_for(n), kBlock, 0, s>>>(qi, pf, cmap.get(), n);
    launched("compose_kernel");
    permute_rows_kernel<<<warp_grid(n), 256, 0, s>>>(op.ro.get(), op.ci.get(), op.v.get(), qf, cmap.get(),
                                                     out->ro.get(), out->ci.get(), out->v.get(), n);
    launched("permute_rows_kernel");
    EW_CUDA_CHECK(cudaStreamSynchronize(s));
    return out;
}

const void* kernel_anchor_order() { return reinterpret_cast<const void*>(&start_kernel); }

}  // namespace ew

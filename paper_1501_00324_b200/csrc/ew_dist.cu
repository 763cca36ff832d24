// Row-partitioned SpMV and Jacobi PCG over several GPUs.
//
// Partition: contiguous row blocks, nnz-balanced (boundary g is the first
// row whose nnz prefix reaches g * nnz / G). Each partition keeps its rows
// with local column numbering: owned columns first (c - r0), then its ghost
// columns in ascending global id (grouped by owner rank, since owners are
// contiguous ranges). Per-row entry order is unchanged, so every row sum of
// the local K1/K2 kernel is the one the single-GPU kernel computes.
//
// Per SpMV: pack the owned values peers need (send lists), exchange them
// into the ghost tail of the extended vector, run the local kernel. Per CG
// reduction: each partition's totals are all-gathered and summed in rank
// order on every rank (deterministic, identical decisions everywhere).
//
// Transports:
//  * peer (one process per GPU, CUDA IPC): every rank maps its peers' ghost
//    buffers and mailboxes; one push kernel gathers the owned values peers
//    need and stores them straight into the peers' ghost tails over NVLink,
//    then raises a flag in each peer's mailbox; dot products are published
//    into every peer's mailbox and summed in rank order. No NCCL on the data
//    path; setup data (ghost requests, IPC handles) goes through the
//    caller's allgather callback. The same kernels run in-process with G
//    partitions on one device (EW_TRANSPORT_PEER with ew_dist_create_peer).
//  * NCCL (one process per GPU; ncclSend/Recv inside a group and
//    ncclAllGather on the caller's stream; libnccl is resolved at run time, so
//    the process uses the same NCCL torch.distributed loaded);
//  * copy: all partitions in this process on the current device, halos as
//    device-to-device copies (tests the partitioned algorithm on 1 GPU).
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>

#include "ew_cg.cuh"

namespace ew {

namespace {

// ---- NCCL, resolved at run time -------------------------------------------
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        // prefer the NCCL already mapped into the process (torch's), then the
        // loader path, then an explicit override
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            if (const char* p = getenv("EW_NCCL_LIBRARY")) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
        }
        if (!h) {
            err = "libnccl.so.2 not found (load torch.distributed first or set EW_NCCL_LIBRARY)";
            return;
        }
        auto sym = [&](const char* n) { return dlsym(h, n); };
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
        api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
        api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
        api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
        api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    });
    if (!api.GetUniqueId || !api.CommInitRank || !api.Send || !api.Recv || !api.AllGather)
        throw Error(EW_UNSUPPORTED, err.empty() ? "NCCL symbols missing" : err);
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw Error(EW_CUDA, std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error"));
}

__global__ void pack_kernel(const int32_t* __restrict__ idx, const double* __restrict__ src, double* __restrict__ dst,
                            int64_t n) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n) dst[k] = src[idx[k]];
}

}  // namespace

// ---- the partition plan (host) ---------------------------------------------
std::vector<int64_t> partition_rows(const int64_t* ro, int64_t nrows, int32_t nparts) {
    require(nparts >= 1, "partition: need at least one part");
    std::vector<int64_t> b(static_cast<size_t>(nparts) + 1, nrows);
    b[0] = 0;
    const int64_t nnz = ro[nrows];
    for (int32_t g = 1; g < nparts; ++g) {
        // first row whose nnz prefix reaches g * nnz / G
        const int64_t target = static_cast<int64_t>((static_cast<__int128>(nnz) * g) / nparts);
        const int64_t* it = std::lower_bound(ro, ro + nrows + 1, target);
        b[g] = std::max<int64_t>(b[g - 1], std::min<int64_t>(nrows, it - ro));
    }
    return b;
}

// A destination of the peer push: send_idx[off, off + cnt) go to the ghost
// tail segment dst_p / dst_x (the peer's p_ext / x_ext) of partition `peer`.
struct PushDesc {
    int64_t off, cnt;
    double* dst_p;
    double* dst_x;
    int32_t peer;
};

// Mailbox words of a partition in a G-way peer transport.
struct Mbox {
    __host__ __device__ static size_t words(int32_t G) { return 7 * static_cast<size_t>(G) + 1; }
    __host__ __device__ static size_t err(int32_t G) { return 7 * static_cast<size_t>(G); }  // a wait timed out
    __host__ __device__ static size_t halo(int32_t g) { return g; }                       // halo epoch raised by g
    __host__ __device__ static size_t ack(int32_t G, int32_t g) { return G + g; }         // g consumed this rank's epoch
    __host__ __device__ static size_t red(int32_t G, int32_t g) { return 2 * G + g; }     // reduction epoch raised by g
    __host__ __device__ static size_t val(int32_t G, int32_t g, uint64_t e) {             // 2 doubles, parity buffered
        return 3 * G + ((e & 1) * G + g) * 2;
    }
};

struct DistPart {
    int32_t part = 0;
    int64_t r0 = 0, r1 = 0, nloc = 0, nghost = 0;
    std::vector<int64_t> recv_off;  // per owner rank, offsets into the ghost tail
    std::vector<int64_t> send_off;  // per peer rank, offsets into send_idx
    DevBuf<int32_t> send_idx;       // local owned indices peers need, grouped by peer
    DevBuf<double> send_buf;
    std::shared_ptr<CsrData> local;
    std::shared_ptr<KernelData> op;
    // Overlap (K1, G > 1): op_int holds the rows without ghost columns and
    // runs while the halo is in flight, op_bnd the rest once it has landed.
    // Both layouts scatter straight into local row ids; op is then unused.
    std::shared_ptr<KernelData> op_int, op_bnd;
    int64_t n_int = 0, n_bnd = 0;
    // CG / SpMV buffers (ext = owned + ghost tail)
    DevBuf<double> x_ext, p_ext, r, q, b, diag, hist, partials, gathered;
    DevBuf<unsigned> tickets;  // SpMV-fused p.q grid sum (cg::grid_sum)
    DevBuf<cg::State> st;
    // peer transport: mailbox (flags + published dot products), push plan
    DevBuf<uint64_t> mbox;
    DevBuf<uint64_t> epochs;  // [0] halo exchanges, [1] reductions completed (device counters)
    DevBuf<unsigned> push_ctr;
    DevBuf<PushDesc> descs;  // one per destination peer
    DevBuf<int32_t> srcs;    // peers that send to this partition
    DevBuf<uint64_t*> mboxes;  // every partition's mailbox, by partition index
    int32_t ndesc = 0, nsrc = 0;
};

struct DistData {
    int32_t nparts = 1, first = 0, nlocal = 1;
    std::vector<int64_t> bounds;
    std::vector<std::unique_ptr<DistPart>> parts;  // this process's partitions
    bool use_nccl = false;
    bool peer = false;                     // peer transport (in-process or CUDA IPC)
    bool ipc = false;                      // peers live in other processes
    std::vector<void*> ipc_mapped;         // cudaIpcOpenMemHandle mappings to close
    ncclComm_t comm = nullptr;
    std::string kernel_id;
    bool split = false;                    // every part has op_int / op_bnd
    cudaStream_t comm_stream = nullptr;    // halo exchange, concurrent with the interior rows
    cudaEvent_t ev_ready = nullptr, ev_halo = nullptr;
    void* hst = nullptr;                   // pinned cg::State[2] for CG polling
    cudaEvent_t poll_ev[2] = {nullptr, nullptr};
    // CG graph of one refresh block (device transports; NCCL runs host-driven)
    cudaStream_t cap = nullptr;
    cudaGraphExec_t exec = nullptr;
    int64_t per_block = 0;
    double g_tol = 0.0, g_div = 0.0;
    int64_t g_interval = -1, g_hist = -1;
    int g_jacobi = -1;
    ~DistData() {
        if (exec) cudaGraphExecDestroy(exec);
        if (cap) cudaStreamDestroy(cap);
        if (hst) cudaFreeHost(hst);
        for (auto e : poll_ev)
            if (e) cudaEventDestroy(e);
        for (void* p : ipc_mapped) cudaIpcCloseMemHandle(p);
        if (ev_ready) cudaEventDestroy(ev_ready);
        if (ev_halo) cudaEventDestroy(ev_halo);
        if (comm_stream) cudaStreamDestroy(comm_stream);
        if (comm) nccl().CommDestroy(comm);
    }
};

namespace {

// ---- peer transport kernels --------------------------------------------------
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ double ld_relaxed_sys(const double* p) {
    double v;
    asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}

// Bounded wait: a peer that never answers (a dead rank) must not hang the
// GPU. After ~30 s of cycles the partition's error word is set, every later
// wait returns at once, and the host reports the failure after the solve.
constexpr long long kSpinLimitCycles = 60'000'000'000ll;

__device__ __forceinline__ void spin_until(const uint64_t* p, uint64_t e, uint64_t* err) {
    if (ld_acquire_sys(err)) return;
    const long long t0 = clock64();
    while (ld_acquire_sys(p) < e) {
        if (clock64() - t0 > kSpinLimitCycles) {
            atomicExch(reinterpret_cast<unsigned long long*>(err), 1ull);
            return;
        }
        __nanosleep(64);
    }
}

// Before a push, every destination must have consumed the previous epoch
// (its ack in this rank's mailbox); with write_acks this rank first acks the
// previous epoch to its own sources (its boundary rows of that epoch are
// done: this kernel is stream-ordered after them). One CTA spins, not the
// push grid: partitions sharing a GPU (or a GPU shared with other work)
// keep their SM slots for the kernels that produce the awaited acks.
__global__ void ack_exchange_kernel(const PushDesc* __restrict__ d, int ndesc, const uint64_t* epochs,
                                    uint64_t* const* mboxes, int me, int G, int write_acks,
                                    const int32_t* __restrict__ srcs, int nsrc) {
    uint64_t* mine = mboxes[me];
    const uint64_t epoch = epochs[0] + 1;  // this exchange (halo_wait_kernel advances the counter)
    if (write_acks)
        for (int i = threadIdx.x; i < nsrc; i += blockDim.x) st_release_sys(mboxes[srcs[i]] + Mbox::ack(G, me), epoch - 1);
    for (int i = threadIdx.x; i < ndesc; i += blockDim.x)
        spin_until(mine + Mbox::ack(G, d[i].peer), epoch - 1, mine + Mbox::err(G));
}

// Pack and transfer in one kernel (after ack_exchange_kernel on the same
// stream): the owned values each destination needs are stored straight into
// its ghost tail (peer stores over NVLink), then the last CTA raises the
// destination's halo flag (release, system scope).
__global__ void push_kernel(const PushDesc* __restrict__ d, int ndesc, const int32_t* __restrict__ idx,
                            const double* __restrict__ src, int which, const uint64_t* epochs, uint64_t* const* mboxes,
                            int me, unsigned* ctr, int64_t total) {
    const uint64_t epoch = epochs[0] + 1;  // this exchange (halo_wait_kernel advances the counter)
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
        int i = 0;
        while (k >= d[i].off + d[i].cnt) ++i;
        double* dst = (which ? d[i].dst_x : d[i].dst_p) + (k - d[i].off);
        *dst = src[idx[k]];
    }
    __threadfence_system();
    __syncthreads();
    __shared__ bool last;
    if (threadIdx.x == 0) last = atomicAdd(ctr, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence_system();
    for (int i = threadIdx.x; i < ndesc; i += blockDim.x) st_release_sys(mboxes[d[i].peer] + Mbox::halo(me), epoch);
    if (threadIdx.x == 0) *ctr = 0;
}

// In-process peer transport: acks as their own launch (every partition's
// boundary rows precede every push on the one device).
__global__ void ack_kernel(uint64_t* const* mboxes, int me, int G, const int32_t* __restrict__ srcs, int nsrc,
                           const uint64_t* epochs) {
    const uint64_t consumed = epochs[0];  // the last exchange this partition finished reading
    for (int i = threadIdx.x; i < nsrc; i += blockDim.x) st_release_sys(mboxes[srcs[i]] + Mbox::ack(G, me), consumed);
}

// The ghost tail is complete once every source raised this epoch.
// Then advances the partition's halo epoch counter (launched once per
// exchange, sources or not).
__global__ void halo_wait_kernel(uint64_t* mine, int G, const int32_t* __restrict__ srcs, int nsrc,
                                 uint64_t* epochs) {
    const uint64_t epoch = epochs[0] + 1;
    for (int i = threadIdx.x; i < nsrc; i += blockDim.x) spin_until(mine + Mbox::halo(srcs[i]), epoch, mine + Mbox::err(G));
    __syncthreads();
    if (threadIdx.x == 0) epochs[0] = epoch;
}

// Reduction, step 1: this partition's totals (State::loc) into slot `me` of
// every partition's mailbox (its own included), then the flag.
__global__ void publish_kernel(const cg::State* st, uint64_t* const* mboxes, int me, int G, const uint64_t* epochs) {
    const uint64_t epoch = epochs[1] + 1;  // this reduction (the collect kernel advances the counter)
    for (int g = threadIdx.x; g < G; g += blockDim.x) {  // any G, not just one warp's worth
        uint64_t* mb = mboxes[g];
        double* v = reinterpret_cast<double*>(mb + Mbox::val(G, me, epoch));
        v[0] = st->loc[0];
        v[1] = st->loc[1];
        __threadfence_system();
        st_release_sys(mb + Mbox::red(G, me), epoch);
    }
}

// Reduction, step 2: wait for every partition's totals, copy them to
// `gathered` in rank order (then cg::finalize_kernel sums them).
__global__ void collect_kernel(uint64_t* mine, int G, uint64_t* epochs, double* gathered) {
    const uint64_t epoch = epochs[1] + 1;
    for (int g = threadIdx.x; g < G; g += blockDim.x) {
        spin_until(mine + Mbox::red(G, g), epoch, mine + Mbox::err(G));
        const double* v = reinterpret_cast<const double*>(mine + Mbox::val(G, g, epoch));
        gathered[2 * g] = ld_relaxed_sys(v);
        gathered[2 * g + 1] = ld_relaxed_sys(v + 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) epochs[1] = epoch;
}

// collect_kernel and cg::finalize_kernel in one launch: thread g waits for
// partition g's totals, thread 0 sums them in rank order and decides.
__global__ void collect_finalize_kernel(uint64_t* mine, int G, uint64_t* epochs, double* gathered, int what,
                                        double tol, double divergence, cg::State* st, double* hist) {
    const uint64_t epoch = epochs[1] + 1;
    for (int g = threadIdx.x; g < G; g += blockDim.x) {
        spin_until(mine + Mbox::red(G, g), epoch, mine + Mbox::err(G));
        const double* v = reinterpret_cast<const double*>(mine + Mbox::val(G, g, epoch));
        gathered[2 * g] = ld_relaxed_sys(v);
        gathered[2 * g + 1] = ld_relaxed_sys(v + 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        epochs[1] = epoch;
        cg::finalize_body(what, gathered, G, tol, divergence, st, hist);
    }
}

// Ghost columns of a row block [r0, r1) given with global column ids:
// sorted, unique, every column outside the block.
std::vector<int64_t> ghost_list(const int64_t* bro, const int64_t* bci, int64_t r0, int64_t r1) {
    std::vector<int64_t> gh;
    const int64_t nloc = r1 - r0;
    for (int64_t k = bro[0]; k < bro[nloc]; ++k)
        if (bci[k] < r0 || bci[k] >= r1) gh.push_back(bci[k]);
    std::sort(gh.begin(), gh.end());
    gh.erase(std::unique(gh.begin(), gh.end()), gh.end());
    return gh;
}

int32_t owner_of(const std::vector<int64_t>& bounds, int64_t c) {
    return static_cast<int32_t>(std::upper_bound(bounds.begin(), bounds.end(), c) - bounds.begin() - 1);
}

// Interior / boundary split for K1 when there is a halo to hide
// (EW_DIST_OVERLAP=0 turns it off for A/B runs).
bool split_rows(const std::string& kid, int32_t G) {
    static const bool on = [] {
        const char* e = std::getenv("EW_DIST_OVERLAP");
        return !(e && e[0] == '0');
    }();
    return on && G > 1 && kid == "k1";
}

// ---- partition build on the device -------------------------------------------
// The block's CSR goes up once; local column numbering, the interior /
// boundary row split and the row subsets are device passes, so the host holds
// nothing beyond the caller's arrays (config 5 on one GPU: 4.5G entries).

// Global -> local column ids: owned c - r0, ghosts nloc + rank in gh (sorted).
__global__ void localize_kernel(const int64_t* __restrict__ cg, int64_t n, int64_t r0, int64_t r1, int64_t nloc,
                                const int64_t* __restrict__ gh, int64_t ngh, int32_t* __restrict__ out, int* bad) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t c = cg[i];
    if (c >= r0 && c < r1) {
        out[i] = static_cast<int32_t>(c - r0);
        return;
    }
    int64_t lo = 0, hi = ngh;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (gh[mid] < c) lo = mid + 1;
        else hi = mid;
    }
    if (lo == ngh || gh[lo] != c) {
        atomicOr(bad, 1);
        out[i] = 0;
        return;
    }
    out[i] = static_cast<int32_t>(nloc + lo);
}

// Row offsets rebased to 0, per-row checks, the longest row and whether a
// row reads a ghost column.
__global__ void local_rows_kernel(int64_t* __restrict__ ro, int64_t base, const int32_t* __restrict__ ci,
                                  int64_t nloc, int64_t nnz, uint8_t* __restrict__ has_ghost, int* maxrow,
                                  int* bad) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= nloc) return;
    const int64_t lo = ro[r] - base, hi = ro[r + 1] - base;
    if (lo > hi || lo < 0 || hi > nnz) {
        atomicOr(bad, 2);
        has_ghost[r] = 0;
        return;
    }
    bool g = false;
    for (int64_t k = lo; k < hi && !g; ++k) g = ci[k] >= nloc;
    has_ghost[r] = g;
    atomicMax(maxrow, static_cast<int>(hi - lo > 0x7fffffff ? 0x7fffffff : hi - lo));
}

__global__ void rebase_kernel(int64_t* __restrict__ ro, int64_t n, int64_t base) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r < n) ro[r] -= base;
}

__global__ void sel_len_kernel(const int64_t* __restrict__ ro, const int32_t* __restrict__ rows, int64_t n,
                               int64_t* __restrict__ len) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) len[i] = ro[rows[i] + 1] - ro[rows[i]];
}

// Entries of the selected rows, one warp per row (coalesced row copies).
__global__ void sel_copy_kernel(const int64_t* __restrict__ ro, const int32_t* __restrict__ ci,
                                const double* __restrict__ v, const int32_t* __restrict__ rows, int64_t n,
                                const int64_t* __restrict__ sro, int32_t* __restrict__ sci, double* __restrict__ sv) {
    const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    const int64_t a = ro[rows[i]], len = ro[rows[i] + 1] - a, d = sro[i];
    for (int64_t k = lane; k < len; k += 32) {
        sci[d + k] = ci[a + k];
        sv[d + k] = v[a + k];
    }
}

// Layout row permutation of a row subset back to local row ids.
__global__ void remap_rows_kernel(int32_t* __restrict__ f, const int32_t* __restrict__ rows, int64_t n) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) f[i] = rows[f[i]];
}

// The block's rows [r0, r1) with local columns: bro = the rows' offsets into
// bci / bv (any base), bci global column ids. has_ghost receives the row flags.
std::shared_ptr<CsrData> upload_local(int64_t nloc, int64_t nghost, const int64_t* bro, const int64_t* bci,
                                      const double* bv, int64_t r0, int64_t r1, const std::vector<int64_t>& ghosts,
                                      DevBuf<uint8_t>& has_ghost, cudaStream_t s) {
    auto m = std::make_shared<CsrData>();
    const int64_t base = bro[0], nnz = bro[nloc] - bro[0];
    require(nnz >= 0, "partition: row offsets decrease");
    m->nrows = nloc;
    m->ncols = nloc + nghost;
    m->nnz = nnz;
    if (m->ncols > 0x7fffffff) throw Error(EW_UNSUPPORTED, "device path supports at most 2^31-1 local columns");
    m->ro.alloc(nloc + 1);
    m->ci.alloc(nnz);
    m->v.alloc(nnz);
    EW_CUDA_CHECK(cudaMemcpyAsync(m->ro.get(), bro, (nloc + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    if (nnz) EW_CUDA_CHECK(cudaMemcpyAsync(m->v.get(), bv + base, nnz * sizeof(double), cudaMemcpyHostToDevice, s));
    DevBuf<int64_t> gh(ghosts.size());
    if (!ghosts.empty())
        EW_CUDA_CHECK(cudaMemcpyAsync(gh.get(), ghosts.data(), ghosts.size() * 8, cudaMemcpyHostToDevice, s));
    Scratch<int> flags(2, s);
    EW_CUDA_CHECK(cudaMemsetAsync(flags.get(), 0, 2 * sizeof(int), s));
    constexpr int64_t kChunk = int64_t{1} << 27;  // 1 GB of int64 column ids per pass
    if (nnz) {
        Scratch<int64_t> cg(std::min(nnz, kChunk), s);
        for (int64_t off = 0; off < nnz; off += kChunk) {
            const int64_t cnt = std::min(kChunk, nnz - off);
            EW_CUDA_CHECK(cudaMemcpyAsync(cg.get(), bci + base + off, cnt * 8, cudaMemcpyHostToDevice, s));
            localize_kernel<<<grid_for(cnt), kBlock, 0, s>>>(cg.get(), cnt, r0, r1, nloc, gh.get(),
                                                             static_cast<int64_t>(ghosts.size()), m->ci.get() + off,
                                                             flags.get());
            launched("localize_kernel");
        }
    }
    has_ghost.alloc(std::max<int64_t>(1, nloc));
    if (nloc) {
        local_rows_kernel<<<grid_for(nloc), kBlock, 0, s>>>(m->ro.get(), base, m->ci.get(), nloc, nnz,
                                                            has_ghost.get(), flags.get() + 1, flags.get());
        launched("local_rows_kernel");
        if (base) {
            rebase_kernel<<<grid_for(nloc + 1), kBlock, 0, s>>>(m->ro.get(), nloc + 1, base);
            launched("rebase_kernel");
        }
    }
    int h[2];
    EW_CUDA_CHECK(cudaMemcpyAsync(h, flags.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
    EW_CUDA_CHECK(cudaStreamSynchronize(s));
    require(!(h[0] & 2), "row_offsets not nondecreasing");
    require(!(h[0] & 1), "partition: a column is neither owned nor in the ghost list");
    m->maxrow = h[1];
    return m;
}

// Rows `rows` (device, ascending local ids) of m as their own CSR.
std::shared_ptr<CsrData> select_rows(const CsrData& m, const int32_t* rows, int64_t n, cudaStream_t s) {
    auto sub = std::make_shared<CsrData>();
    sub->nrows = n;
    sub->ncols = m.ncols;
    sub->maxrow = m.maxrow;
    sub->ro.alloc(n + 1);
    EW_CUDA_CHECK(cudaMemsetAsync(sub->ro.get(), 0, sizeof(int64_t), s));
    if (n) {
        Scratch<int64_t> len(n, s);
        sel_len_kernel<<<grid_for(n), kBlock, 0, s>>>(m.ro.get(), rows, n, len.get());
        launched("sel_len_kernel");
        size_t bytes = 0;
        EW_CUDA_CHECK(cub::DeviceScan::InclusiveSum(nullptr, bytes, len.get(), sub->ro.get() + 1, n, s));
        Scratch<unsigned char> tmp(bytes, s);
        EW_CUDA_CHECK(cub::DeviceScan::InclusiveSum(tmp.get(), bytes, len.get(), sub->ro.get() + 1, n, s));
        launched("cub::DeviceScan::InclusiveSum");
    }
    EW_CUDA_CHECK(cudaMemcpyAsync(&sub->nnz, sub->ro.get() + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    EW_CUDA_CHECK(cudaStreamSynchronize(s));
    sub->ci.alloc(sub->nnz);
    sub->v.alloc(sub->nnz);
    if (n) {
        sel_copy_kernel<<<grid_for(n * 32), kBlock, 0, s>>>(m.ro.get(), m.ci.get(), m.v.get(), rows, n,
                                                            sub->ro.get(), sub->ci.get(), sub->v.get());
        launched("sel_copy_kernel");
    }
    return sub;
}

// ids[i] = i; flag[i] = has_ghost[i] == want
__global__ void row_sel_kernel(const uint8_t* __restrict__ has_ghost, int64_t n, uint8_t want,
                               int32_t* __restrict__ ids, uint8_t* __restrict__ flag) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    ids[i] = static_cast<int32_t>(i);
    flag[i] = (has_ghost[i] != 0) == (want != 0);
}

// Local row ids with has_ghost == want (ascending), on the device.
int64_t flagged_rows(const DevBuf<uint8_t>& has_ghost, int64_t nloc, bool want, DevBuf<int32_t>& out, cudaStream_t s) {
    out.alloc(std::max<int64_t>(1, nloc));
    if (!nloc) return 0;
    Scratch<int64_t> cnt(1, s);
    Scratch<int32_t> ids(nloc, s);
    Scratch<uint8_t> flag(nloc, s);
    row_sel_kernel<<<grid_for(nloc), kBlock, 0, s>>>(has_ghost.get(), nloc, want ? 1 : 0, ids.get(), flag.get());
    launched("row_sel_kernel");
    size_t bytes = 0;
    EW_CUDA_CHECK(cub::DeviceSelect::Flagged(nullptr, bytes, ids.get(), flag.get(), out.get(), cnt.get(), nloc, s));
    Scratch<unsigned char> tmp(bytes, s);
    EW_CUDA_CHECK(cub::DeviceSelect::Flagged(tmp.get(), bytes, ids.get(), flag.get(), out.get(), cnt.get(), nloc, s));
    launched("cub::DeviceSelect::Flagged");
    int64_t n = 0;
    EW_CUDA_CHECK(cudaMemcpyAsync(&n, cnt.get(), sizeof(n), cudaMemcpyDeviceToHost, s));
    EW_CUDA_CHECK(cudaStreamSynchronize(s));
    return n;
}

// K1 kernel over the local rows `rows` (device, ascending), entries in their
// order, its layout scattering into local row ids.
std::shared_ptr<KernelData> prepare_rows(const CsrData& local, const DevBuf<int32_t>& rows, int64_t n,
                                         const std::string& kid, const ew_warp_config& cfg,
                                         const ew_kernel_options& opts, cudaStream_t s) {
    std::shared_ptr<KernelData> k;
    {
        auto sub = select_rows(local, rows.get(), n, s);
        k = prepare(kid, *sub, cfg, opts, s);
        EW_CUDA_CHECK(cudaStreamSynchronize(s));
    }
    if (n) {
        remap_rows_kernel<<<grid_for(n), kBlock, 0, s>>>(k->layout->fwd.get(), rows.get(), n);
        launched("remap_rows_kernel");
        EW_CUDA_CHECK(cudaStreamSynchronize(s));
    }
    return k;
}

// Partition g from its row block (bro: the rows' offsets into bci / bv,
// bci: global column ids, bv: values), its ghost list and, per peer, the
// global ids that peer needs from this partition (ascending).
void build_part(DistPart& P, int32_t g, int32_t G, const std::vector<int64_t>& bounds, const int64_t* bro,
                const int64_t* bci, const double* bv, const std::vector<int64_t>& ghosts,
                const std::vector<std::vector<int64_t>>& peer_needs, const std::string& kid,
                const ew_warp_config& cfg, const ew_kernel_options& opts, cudaStream_t s) {
    load_all_kernels();  // before any exchange: no lazy load while a peer spins
    P.part = g;
    P.r0 = bounds[g];
    P.r1 = bounds[g + 1];
    P.nloc = P.r1 - P.r0;
    P.nghost = static_cast<int64_t>(ghosts.size());
    P.recv_off.assign(G + 1, 0);
    for (int64_t c : ghosts) P.recv_off[owner_of(bounds, c) + 1]++;
    for (int32_t h = 0; h < G; ++h) P.recv_off[h + 1] += P.recv_off[h];
    std::vector<int32_t> sidx;
    P.send_off.assign(G + 1, 0);
    for (int32_t h = 0; h < G; ++h) {
        for (int64_t c : peer_needs[h]) {
            require(c >= P.r0 && c < P.r1, "partition: a peer requested a row this partition does not own");
            sidx.push_back(static_cast<int32_t>(c - P.r0));
        }
        P.send_off[h + 1] = static_cast<int64_t>(sidx.size());
    }
    // local CSR on the device: owned columns c - r0, ghosts nloc + their
    // position in `ghosts`
    DevBuf<uint8_t> has_ghost;
    auto local = upload_local(P.nloc, P.nghost, bro, bci, bv, P.r0, P.r1, ghosts, has_ghost, s);
    if (split_rows(kid, G)) {
        DevBuf<int32_t> rows_int, rows_bnd;
        P.n_int = flagged_rows(has_ghost, P.nloc, false, rows_int, s);
        P.n_bnd = flagged_rows(has_ghost, P.nloc, true, rows_bnd, s);
        has_ghost.release();
        P.op_int = prepare_rows(*local, rows_int, P.n_int, kid, cfg, opts, s);
        P.op_bnd = prepare_rows(*local, rows_bnd, P.n_bnd, kid, cfg, opts, s);
        // the boundary rows run the split-x K1, which reads the int32 slab
        if (P.op_bnd->layout) restore_columns(*P.op_bnd->layout, s);
    } else {
        has_ghost.release();
        P.op = prepare(kid, *local, cfg, opts, s);
        // the K1 / K2 layout holds its own copy of the entries; other kernel
        // kinds keep referring to the local CSR
        if (kid != "k1" && kid != "k2") P.local = local;
    }
    EW_CUDA_CHECK(cudaStreamSynchronize(s));
    local.reset();
    P.send_idx.alloc(sidx.size());
    P.send_buf.alloc(sidx.size());
    if (!sidx.empty())
        EW_CUDA_CHECK(cudaMemcpyAsync(P.send_idx.get(), sidx.data(), sidx.size() * 4, cudaMemcpyHostToDevice, s));
    P.x_ext.alloc(P.nloc + P.nghost);
    P.p_ext.alloc(P.nloc + P.nghost);
    P.q.alloc(P.nloc);
    P.gathered.alloc(2 * static_cast<size_t>(G));
    EW_CUDA_CHECK(cudaStreamSynchronize(s));
}

// Peer transport, first half: push this epoch's values into the peers'
// ghost tails (on stream s). which: 0 p_ext, 1 x_ext.
// Owned values come from `src` (per local partition) when given, else from
// the owned part of ext.
using PartPtrs = std::vector<const double*>;

void peer_push(DistData& D, int which, DevBuf<double> DistPart::*ext, cudaStream_t s, const PartPtrs* src = nullptr) {
    const int32_t G = D.nparts;
    if (!D.ipc) {
        for (auto& P : D.parts) {
            if (!P->nsrc) continue;
            ack_kernel<<<1, 32, 0, s>>>(P->mboxes.get(), P->part, G, P->srcs.get(), P->nsrc, P->epochs.get());
            launched("ack_kernel");
        }
    }
    for (size_t i = 0; i < D.parts.size(); ++i) {
        auto& P = D.parts[i];
        const int64_t total = static_cast<int64_t>(P->send_idx.size());
        if (!total && (!D.ipc || !P->nsrc)) continue;
        const unsigned grid = std::max<unsigned>(1, std::min<unsigned>(grid_for(total), 148 * 4));
        const double* from = src ? (*src)[i] : ((*P).*ext).get();
        ack_exchange_kernel<<<1, 32, 0, s>>>(P->descs.get(), P->ndesc, P->epochs.get(), P->mboxes.get(), P->part, G,
                                             D.ipc ? 1 : 0, P->srcs.get(), P->nsrc);
        launched("ack_exchange_kernel");
        push_kernel<<<grid, kBlock, 0, s>>>(P->descs.get(), P->ndesc, P->send_idx.get(), from, which, P->epochs.get(),
                                            P->mboxes.get(), P->part, P->push_ctr.get(), total);
        launched("push_kernel");
    }
}

// Peer transport, second half: on stream s, wait until every ghost of this
// epoch has landed.
void peer_wait(DistData& D, cudaStream_t s) {
    for (auto& P : D.parts) {
        halo_wait_kernel<<<1, 32, 0, s>>>(P->mbox.get(), D.nparts, P->srcs.get(), P->nsrc, P->epochs.get());
        launched("halo_wait_kernel");
    }
}

// Exchange the owned values peers need into every partition's ghost tail.
void halo(DistData& D, DevBuf<double> DistPart::*ext, cudaStream_t s, const PartPtrs* src = nullptr) {
    const int32_t G = D.nparts;
    if (G == 1) return;
    if (D.peer) {
        peer_push(D, ext == &DistPart::x_ext ? 1 : 0, ext, s, src);
        peer_wait(D, s);
        return;
    }
    for (size_t i = 0; i < D.parts.size(); ++i) {
        auto& P = D.parts[i];
        const int64_t ns = static_cast<int64_t>(P->send_idx.size());
        if (ns) {
            const double* from = src ? (*src)[i] : ((*P).*ext).get();
            pack_kernel<<<grid_for(ns), kBlock, 0, s>>>(P->send_idx.get(), from, P->send_buf.get(), ns);
            launched("pack_kernel");
        }
    }
    if (D.use_nccl) {
        DistPart& P = *D.parts[0];
        const auto& api = nccl();
        nccl_check(api.GroupStart(), "ncclGroupStart");
        for (int32_t h = 0; h < G; ++h) {
            if (h == P.part) continue;
            const int64_t sc = P.send_off[h + 1] - P.send_off[h];
            const int64_t rc = P.recv_off[h + 1] - P.recv_off[h];
            if (sc) nccl_check(api.Send(P.send_buf.get() + P.send_off[h], sc, ncclFloat64, h, D.comm, s), "ncclSend");
            if (rc)
                nccl_check(api.Recv((P.*ext).get() + P.nloc + P.recv_off[h], rc, ncclFloat64, h, D.comm, s),
                           "ncclRecv");
        }
        nccl_check(api.GroupEnd(), "ncclGroupEnd");
        return;
    }
    // in-process: partition h's segment for g lands in g's ghost tail
    for (auto& Pg : D.parts) {
        for (auto& Ph : D.parts) {
            if (Ph->part == Pg->part) continue;
            const int64_t rc = Pg->recv_off[Ph->part + 1] - Pg->recv_off[Ph->part];
            if (!rc) continue;
            EW_CUDA_CHECK(cudaMemcpyAsync(((*Pg).*ext).get() + Pg->nloc + Pg->recv_off[Ph->part],
                                          Ph->send_buf.get() + Ph->send_off[Pg->part], rc * 8,
                                          cudaMemcpyDeviceToDevice, s));
        }
    }
}

// Every partition's State::loc[0..1] into every partition's `gathered`.
void allgather(DistData& D, cudaStream_t s) {
    if (D.peer) {
        for (auto& P : D.parts) {
            publish_kernel<<<1, 32, 0, s>>>(P->st.get(), P->mboxes.get(), P->part, D.nparts, P->epochs.get());
            launched("publish_kernel");
        }
        for (auto& P : D.parts) {
            collect_kernel<<<1, 32, 0, s>>>(P->mbox.get(), D.nparts, P->epochs.get(), P->gathered.get());
            launched("collect_kernel");
        }
        return;
    }
    if (D.use_nccl) {
        DistPart& P = *D.parts[0];
        nccl_check(nccl().AllGather(P.st.get()->loc, P.gathered.get(), 2, ncclFloat64, D.comm, s), "ncclAllGather");
        return;
    }
    for (auto& Pg : D.parts)
        for (auto& Ph : D.parts)
            EW_CUDA_CHECK(cudaMemcpyAsync(Pg->gathered.get() + 2 * Ph->part, Ph->st.get()->loc, 16,
                                          cudaMemcpyDeviceToDevice, s));
}

void finalize(DistData& D, int what, const ew_cg_config& cfg, cudaStream_t s) {
    for (auto& P : D.parts) {
        cg::finalize_kernel<<<1, 1, 0, s>>>(what, P->gathered.get(), D.nparts, cfg.rel_tolerance,
                                            cfg.divergence_limit, P->st.get(), P->hist.get());
        launched("cg::finalize_kernel");
    }
}

// A CG reduction: every partition's State::loc totals summed in rank order on
// every partition, then the reference's decision.
void reduce_finalize(DistData& D, int what, const ew_cg_config& cfg, cudaStream_t s) {
    if (!D.peer) {
        allgather(D, s);
        finalize(D, what, cfg, s);
        return;
    }
    for (auto& P : D.parts) {
        publish_kernel<<<1, 32, 0, s>>>(P->st.get(), P->mboxes.get(), P->part, D.nparts, P->epochs.get());
        launched("publish_kernel");
    }
    for (auto& P : D.parts) {
        collect_finalize_kernel<<<1, 32, 0, s>>>(P->mbox.get(), D.nparts, P->epochs.get(), P->gathered.get(), what,
                                                 cfg.rel_tolerance, cfg.divergence_limit, P->st.get(),
                                                 P->hist.get());
        launched("collect_finalize_kernel");
    }
}

// The exchange on the comm stream, ordered after everything already on s.
void halo_begin(DistData& D, DevBuf<double> DistPart::*ext, cudaStream_t s, const PartPtrs* src = nullptr) {
    EW_CUDA_CHECK(cudaEventRecord(D.ev_ready, s));
    EW_CUDA_CHECK(cudaStreamWaitEvent(D.comm_stream, D.ev_ready, 0));
    if (D.peer) {  // the push runs beside the interior rows; peer_wait orders the boundary rows
        peer_push(D, ext == &DistPart::x_ext ? 1 : 0, ext, D.comm_stream, src);
        return;
    }
    halo(D, ext, D.comm_stream, src);
    EW_CUDA_CHECK(cudaEventRecord(D.ev_halo, D.comm_stream));
}

void halo_end(DistData& D, cudaStream_t s) {
    if (D.peer) {
        peer_wait(D, s);
        // the push kernels read p_ext / x_ext: the next writer (p update) on s
        // must not overtake them
        EW_CUDA_CHECK(cudaEventRecord(D.ev_halo, D.comm_stream));
    }
    EW_CUDA_CHECK(cudaStreamWaitEvent(s, D.ev_halo, 0));
}

// One row set of a split part; with `dot`, its p.q partial goes to loc[slot].
// False when the fused dot was not available (the caller runs pq_kernel).
bool run_rows(DistPart& P, const KernelData& k, int64_t nrows, int slot, const double* xe, cudaStream_t s,
              const int* done, bool dot, double* y = nullptr) {
    if (!nrows) {
        if (dot) EW_CUDA_CHECK(cudaMemsetAsync(P.st.get()->loc + slot, 0, (slot == 0 ? 2 : 1) * sizeof(double), s));
        return true;
    }
    if (dot && kernel_apply_dot(k, xe, P.q.get(), false, s, done,
                                DotSink{P.partials.get(), static_cast<unsigned>(P.partials.size()), P.tickets.get(),
                                        P.st.get(), 1, slot}))
        return true;
    kernel_apply(k, xe, y ? y : P.q.get(), false, s, done);
    return !dot;
}

// q = A x_ext on every local partition after (or, split, overlapped with)
// the halo exchange of `ext`; dot: p.q into each part's State::loc.
// xs / ys (split parts, no dot): the caller's owned x and y per partition;
// the owned x is read in place (interior rows directly, boundary rows with
// the split-x kernel) and y written in place: only the ghosts go to ext.
void spmv_exchange(DistData& D, DevBuf<double> DistPart::*ext, cudaStream_t s, bool guard, bool dot,
                   bool exchange = true, const PartPtrs* xs = nullptr, const std::vector<double*>* ys = nullptr) {
    std::vector<char> fused(D.parts.size(), 1);
    if (!D.split) {
        if (exchange) halo(D, ext, s);
        for (size_t i = 0; i < D.parts.size(); ++i) {
            DistPart& P = *D.parts[i];
            fused[i] = run_rows(P, *P.op, P.nloc, 0, ((P).*ext).get(), s, guard ? &P.st.get()->done : nullptr, dot);
        }
    } else {
        if (exchange) halo_begin(D, ext, s, xs);
        for (size_t i = 0; i < D.parts.size(); ++i) {
            DistPart& P = *D.parts[i];
            fused[i] = run_rows(P, *P.op_int, P.n_int, 0, xs ? (*xs)[i] : ((P).*ext).get(), s,
                                guard ? &P.st.get()->done : nullptr, dot, ys ? (*ys)[i] : nullptr);
        }
        if (exchange) halo_end(D, s);
        for (size_t i = 0; i < D.parts.size(); ++i) {
            DistPart& P = *D.parts[i];
            if (xs) {
                if (P.n_bnd)
                    layout_spmv_split(*P.op_bnd->layout, (*xs)[i], ((P).*ext).get() + P.nloc, P.nloc, (*ys)[i], s);
                continue;
            }
            fused[i] &= run_rows(P, *P.op_bnd, P.n_bnd, 1, ((P).*ext).get(), s, guard ? &P.st.get()->done : nullptr,
                                 dot);
        }
    }
    if (!dot) return;
    for (size_t i = 0; i < D.parts.size(); ++i) {
        if (fused[i]) continue;
        DistPart& P = *D.parts[i];
        cg::pq_kernel<true><<<cg::red_grid(P.nloc), cg::kRedBlock, 0, s>>>(((P).*ext).get(), P.q.get(), P.nloc,
                                                                          P.partials.get(), P.st.get());
        launched("cg::pq_kernel<dist>");
    }
}

// Peer plan of partition P: its mailbox, sources, and one push descriptor
// per destination h (the ghost segment h keeps for P's values starts at
// h's nloc + h's recv_off[P]). peer_p/x/mbox/nloc/recv index partitions.
void peer_plan(DistPart& P, int32_t G, const std::vector<double*>& peer_p, const std::vector<double*>& peer_x,
               const std::vector<uint64_t*>& mbox, const std::vector<int64_t>& tail_off, cudaStream_t s) {
    std::vector<PushDesc> d;
    for (int32_t h = 0; h < G; ++h) {
        const int64_t cnt = P.send_off[h + 1] - P.send_off[h];
        if (h == P.part || !cnt) continue;
        d.push_back(PushDesc{P.send_off[h], cnt, peer_p[h] + tail_off[h], peer_x[h] + tail_off[h], h});
    }
    std::vector<int32_t> src;
    for (int32_t h = 0; h < G; ++h)
        if (h != P.part && P.recv_off[h + 1] > P.recv_off[h]) src.push_back(h);
    P.ndesc = static_cast<int32_t>(d.size());
    P.nsrc = static_cast<int32_t>(src.size());
    P.descs.alloc(std::max<size_t>(1, d.size()));
    P.srcs.alloc(std::max<size_t>(1, src.size()));
    P.mboxes.alloc(G);
    if (!d.empty())
        EW_CUDA_CHECK(cudaMemcpyAsync(P.descs.get(), d.data(), d.size() * sizeof(PushDesc), cudaMemcpyHostToDevice, s));
    if (!src.empty())
        EW_CUDA_CHECK(cudaMemcpyAsync(P.srcs.get(), src.data(), src.size() * 4, cudaMemcpyHostToDevice, s));
    EW_CUDA_CHECK(cudaMemcpyAsync(P.mboxes.get(), mbox.data(), G * sizeof(uint64_t*), cudaMemcpyHostToDevice, s));
    EW_CUDA_CHECK(cudaStreamSynchronize(s));
}

void alloc_mailbox(DistPart& P, int32_t G, cudaStream_t s) {
    P.mbox.alloc(Mbox::words(G));
    P.epochs.alloc(2);
    EW_CUDA_CHECK(cudaMemsetAsync(P.epochs.get(), 0, P.epochs.bytes(), s));
    P.push_ctr.alloc(1);
    EW_CUDA_CHECK(cudaMemsetAsync(P.mbox.get(), 0, P.mbox.bytes(), s));
    EW_CUDA_CHECK(cudaMemsetAsync(P.push_ctr.get(), 0, P.push_ctr.bytes(), s));
}

// In-process peer transport: the "peers" are this process's partitions.
void peer_setup_local(DistData& D, cudaStream_t s) {
    const int32_t G = D.nparts;
    for (auto& P : D.parts) alloc_mailbox(*P, G, s);
    std::vector<double*> pp(G), px(G);
    std::vector<uint64_t*> mb(G);
    for (auto& P : D.parts) {
        pp[P->part] = P->p_ext.get();
        px[P->part] = P->x_ext.get();
        mb[P->part] = P->mbox.get();
    }
    for (auto& P : D.parts) {
        std::vector<int64_t> tail(G, 0);
        for (auto& H : D.parts)
            if (H->part != P->part) tail[H->part] = H->nloc + H->recv_off[P->part];
        peer_plan(*P, G, pp, px, mb, tail, s);
    }
    D.peer = true;
}

void init_overlap(DistData& D) {
    D.split = !D.parts.empty();
    for (auto& P : D.parts) D.split = D.split && P->op_int && P->op_bnd;
    if (!D.split) return;
    EW_CUDA_CHECK(cudaStreamCreateWithFlags(&D.comm_stream, cudaStreamNonBlocking));
    EW_CUDA_CHECK(cudaEventCreateWithFlags(&D.ev_ready, cudaEventDisableTiming));
    EW_CUDA_CHECK(cudaEventCreateWithFlags(&D.ev_halo, cudaEventDisableTiming));
}

}  // namespace

std::shared_ptr<DistData> dist_create(int64_t nrows, int64_t ncols, const int64_t* ro, const int64_t* ci,
                                      const double* v, const int64_t* bounds_in, int32_t nparts, int32_t first,
                                      int32_t nlocal, const void* nccl_id, const std::string& kid,
                                      const ew_warp_config& cfg, const ew_kernel_options& opts, cudaStream_t s,
                                      bool peer) {
    require(nrows == ncols, "partitioned operator must be square");
    require(nparts >= 1 && first >= 0 && nlocal >= 1 && first + nlocal <= nparts, "bad partition range");
    require(kid == "k1" || kid == "k2" || kid == "csr_ref" || kid == "csr_vector" || kid == "ell" || kid == "hyb" ||
                kid == "coo",
            "partitioned kernels: the local matrix is rectangular (ghost columns), so r/rs ids do not apply");
    auto D = std::make_shared<DistData>();
    D->nparts = nparts;
    D->first = first;
    D->nlocal = nlocal;
    D->kernel_id = kid;
    D->bounds = bounds_in ? std::vector<int64_t>(bounds_in, bounds_in + nparts + 1) : partition_rows(ro, nrows, nparts);
    require(D->bounds.front() == 0 && D->bounds.back() == nrows, "partition bounds must cover [0, nrows]");
    for (int32_t g = 0; g < nparts; ++g) require(D->bounds[g] <= D->bounds[g + 1], "partition bounds must be sorted");
    D->use_nccl = nccl_id != nullptr;
    if (D->use_nccl) {
        require(nlocal == 1, "the NCCL transport runs one partition per process");
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof(id));
        nccl_check(nccl().CommInitRank(&D->comm, nparts, id, first), "ncclCommInitRank");
    } else {
        require(nlocal == nparts, "the in-process transport holds every partition");
    }
    // every partition's ghost list is computable from the global CSR
    std::vector<std::vector<int64_t>> ghosts(nparts);
    for (int32_t h = 0; h < nparts; ++h)
        ghosts[h] = ghost_list(ro + D->bounds[h], ci, D->bounds[h], D->bounds[h + 1]);
    for (int32_t g = first; g < first + nlocal; ++g) {
        std::vector<std::vector<int64_t>> needs(nparts);
        for (int32_t h = 0; h < nparts; ++h) {
            if (h == g) continue;
            for (int64_t c : ghosts[h])
                if (c >= D->bounds[g] && c < D->bounds[g + 1]) needs[h].push_back(c);
        }
        auto P = std::make_unique<DistPart>();
        build_part(*P, g, nparts, D->bounds, ro + D->bounds[g], ci, v, ghosts[g], needs, kid, cfg, opts, s);
        D->parts.push_back(std::move(P));
    }
    if (peer) {
        require(!D->use_nccl, "the in-process peer transport holds every partition");
        if (nparts > 1) peer_setup_local(*D, s);
    }
    init_overlap(*D);
    return D;
}

std::shared_ptr<DistData> dist_create_block(int64_t nglobal, const int64_t* bro, const int64_t* bci,
                                            const double* bv, const int64_t* bounds, int32_t nparts, int32_t rank,
                                            const void* nccl_id, const std::string& kid, const ew_warp_config& cfg,
                                            const ew_kernel_options& opts, cudaStream_t s) {
    require(nccl_id != nullptr, "the block constructor needs the NCCL transport");
    require(nparts >= 1 && rank >= 0 && rank < nparts, "bad rank");
    require(kid == "k1" || kid == "k2" || kid == "csr_ref",
            "partitioned kernels: k1, k2 or csr_ref (the local matrix has ghost columns)");
    auto D = std::make_shared<DistData>();
    D->nparts = nparts;
    D->first = rank;
    D->nlocal = 1;
    D->kernel_id = kid;
    D->bounds.assign(bounds, bounds + nparts + 1);
    require(D->bounds.front() == 0 && D->bounds.back() == nglobal, "partition bounds must cover [0, nrows]");
    for (int32_t g = 0; g < nparts; ++g) require(D->bounds[g] <= D->bounds[g + 1], "partition bounds must be sorted");
    D->use_nccl = true;
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    const auto& api = nccl();
    nccl_check(api.CommInitRank(&D->comm, nparts, id, rank), "ncclCommInitRank");
    const int64_t r0 = D->bounds[rank], r1 = D->bounds[rank + 1];
    const std::vector<int64_t> ghosts = ghost_list(bro, bci, r0, r1);
    // setup exchange: how many ghosts each rank needs from each owner, then
    // the ghost ids themselves (owner-grouped, ascending)
    std::vector<int64_t> my_need(nparts, 0);
    for (int64_t c : ghosts) my_need[owner_of(D->bounds, c)]++;
    std::vector<std::vector<int64_t>> needs(nparts);
    {
        DevBuf<int64_t> dneed(nparts), dall(static_cast<size_t>(nparts) * nparts);
        EW_CUDA_CHECK(cudaMemcpyAsync(dneed.get(), my_need.data(), nparts * 8, cudaMemcpyHostToDevice, s));
        nccl_check(api.AllGather(dneed.get(), dall.get(), nparts, ncclInt64, D->comm, s), "ncclAllGather(needs)");
        std::vector<int64_t> all(static_cast<size_t>(nparts) * nparts);
        EW_CUDA_CHECK(cudaMemcpyAsync(all.data(), dall.get(), all.size() * 8, cudaMemcpyDeviceToHost, s));
        EW_CUDA_CHECK(cudaStreamSynchronize(s));
        std::vector<int64_t> goff(nparts + 1, 0);
        for (int32_t h = 0; h < nparts; ++h) goff[h + 1] = goff[h] + my_need[h];
        int64_t total_in = 0;
        for (int32_t h = 0; h < nparts; ++h) total_in += all[static_cast<size_t>(h) * nparts + rank];
        DevBuf<int64_t> dgh(ghosts.size()), din(total_in);
        if (!ghosts.empty())
            EW_CUDA_CHECK(cudaMemcpyAsync(dgh.get(), ghosts.data(), ghosts.size() * 8, cudaMemcpyHostToDevice, s));
        nccl_check(api.GroupStart(), "ncclGroupStart");
        int64_t in_off = 0;
        std::vector<int64_t> ioff(nparts + 1, 0);
        for (int32_t h = 0; h < nparts; ++h) {
            const int64_t cnt_in = all[static_cast<size_t>(h) * nparts + rank];
            ioff[h] = in_off;
            if (h != rank) {
                if (my_need[h]) nccl_check(api.Send(dgh.get() + goff[h], my_need[h], ncclInt64, h, D->comm, s), "ncclSend");
                if (cnt_in) nccl_check(api.Recv(din.get() + in_off, cnt_in, ncclInt64, h, D->comm, s), "ncclRecv");
            }
            in_off += cnt_in;
        }
        ioff[nparts] = in_off;
        nccl_check(api.GroupEnd(), "ncclGroupEnd");
        std::vector<int64_t> hin(total_in);
        if (total_in) EW_CUDA_CHECK(cudaMemcpyAsync(hin.data(), din.get(), total_in * 8, cudaMemcpyDeviceToHost, s));
        EW_CUDA_CHECK(cudaStreamSynchronize(s));
        for (int32_t h = 0; h < nparts; ++h)
            if (h != rank) needs[h].assign(hin.begin() + ioff[h], hin.begin() + ioff[h + 1]);
    }
    auto P = std::make_unique<DistPart>();
    build_part(*P, rank, nparts, D->bounds, bro, bci, bv, ghosts, needs, kid, cfg, opts, s);
    D->parts.push_back(std::move(P));
    init_overlap(*D);
    return D;
}

// The setup exchange of one rank's row block (host only, the caller's
// allgather): its ghost list (columns outside the block, ascending, so
// grouped by owner) and, per peer, the global rows that peer needs from this
// block (ascending). counts[h * G + g]: how many of h's ghosts g owns.
BlockPlan block_plan(int64_t nloc, const int64_t* bro, const int64_t* bci, const std::vector<int64_t>& bounds,
                     int32_t rank, ew_allgather_fn allgather, void* user) {
    const int32_t G = static_cast<int32_t>(bounds.size()) - 1;
    require(G >= 1 && rank >= 0 && rank < G, "bad rank");
    require(bounds[rank + 1] - bounds[rank] == nloc, "row block does not match the bounds");
    auto ag = [&](const void* send, void* recv, size_t bytes) {
        if (allgather(send, recv, bytes, user) != 0) throw Error(EW_INVALID_ARGUMENT, "allgather callback failed");
    };
    const int64_t r0 = bounds[rank], r1 = bounds[rank + 1];
    const int64_t nglobal = bounds[G];
    for (int64_t k = bro[0]; k < bro[nloc]; ++k)
        require(bci[k] >= 0 && bci[k] < nglobal, "column out of range");
    BlockPlan plan;
    plan.ghosts = ghost_list(bro, bci, r0, r1);
    // ghost requests: counts per owner, then the (owner-grouped, ascending) ids
    std::vector<int64_t> my_need(G, 0);
    plan.counts.assign(static_cast<size_t>(G) * G, 0);
    for (int64_t c : plan.ghosts) my_need[owner_of(bounds, c)]++;
    ag(my_need.data(), plan.counts.data(), G * sizeof(int64_t));
    int64_t maxg = 1;
    for (int32_t h = 0; h < G; ++h) {
        int64_t t = 0;
        for (int32_t g = 0; g < G; ++g) t += plan.counts[static_cast<size_t>(h) * G + g];
        maxg = std::max(maxg, t);
    }
    std::vector<int64_t> mine(maxg, -1), every(static_cast<size_t>(G) * maxg);
    std::copy(plan.ghosts.begin(), plan.ghosts.end(), mine.begin());
    ag(mine.data(), every.data(), maxg * sizeof(int64_t));
    plan.needs.assign(G, {});
    for (int32_t h = 0; h < G; ++h) {
        if (h == rank) continue;
        int64_t skip = 0;  // h's ghosts owned by ranks < rank
        for (int32_t g = 0; g < rank; ++g) skip += plan.counts[static_cast<size_t>(h) * G + g];
        const int64_t* lst = every.data() + static_cast<size_t>(h) * maxg + skip;
        plan.needs[h].assign(lst, lst + plan.counts[static_cast<size_t>(h) * G + rank]);
    }
    return plan;
}

std::shared_ptr<DistData> dist_create_block_ipc(int64_t nglobal, const int64_t* bro, const int64_t* bci,
                                                const double* bv, const int64_t* bounds, int32_t nparts,
                                                int32_t rank, ew_allgather_fn allgather, void* user,
                                                const std::string& kid, const ew_warp_config& cfg,
                                                const ew_kernel_options& opts, cudaStream_t s) {
    require(allgather != nullptr, "the IPC transport needs an allgather callback");
    require(nparts >= 1 && rank >= 0 && rank < nparts, "bad rank");
    require(kid == "k1" || kid == "k2" || kid == "csr_ref",
            "partitioned kernels: k1, k2 or csr_ref (the local matrix has ghost columns)");
    auto D = std::make_shared<DistData>();
    D->nparts = nparts;
    D->first = rank;
    D->nlocal = 1;
    D->kernel_id = kid;
    D->bounds.assign(bounds, bounds + nparts + 1);
    require(D->bounds.front() == 0 && D->bounds.back() == nglobal, "partition bounds must cover [0, nrows]");
    for (int32_t g = 0; g < nparts; ++g) require(D->bounds[g] <= D->bounds[g + 1], "partition bounds must be sorted");
    const int32_t G = nparts;
    auto ag = [&](const void* send, void* recv, size_t bytes) {
        if (allgather(send, recv, bytes, user) != 0) throw Error(EW_INVALID_ARGUMENT, "allgather callback failed");
    };
    const int64_t nloc = D->bounds[rank + 1] - D->bounds[rank];
    BlockPlan plan = block_plan(nloc, bro, bci, D->bounds, rank, allgather, user);
    const std::vector<int64_t>& ghosts = plan.ghosts;
    const std::vector<std::vector<int64_t>>& needs = plan.needs;
    auto before = [&](int32_t h, int32_t owner) {  // h's ghosts owned by ranks < owner
        int64_t t = 0;
        for (int32_t g = 0; g < owner; ++g) t += plan.counts[static_cast<size_t>(h) * G + g];
        return t;
    };
    auto P = std::make_unique<DistPart>();
    build_part(*P, rank, nparts, D->bounds, bro, bci, bv, ghosts, needs, kid, cfg, opts, s);
    if (G > 1) {
        require(P->nloc > 0, "the IPC transport needs at least one row per rank");
        alloc_mailbox(*P, G, s);
        struct Ex {
            cudaIpcMemHandle_t p, x, mb;
        } ex{}, *exs = nullptr;
        EW_CUDA_CHECK(cudaIpcGetMemHandle(&ex.p, P->p_ext.get()));
        EW_CUDA_CHECK(cudaIpcGetMemHandle(&ex.x, P->x_ext.get()));
        EW_CUDA_CHECK(cudaIpcGetMemHandle(&ex.mb, P->mbox.get()));
        std::vector<Ex> all_ex(G);
        exs = all_ex.data();
        ag(&ex, exs, sizeof(Ex));
        std::vector<double*> pp(G), px(G);
        std::vector<uint64_t*> mb(G);
        std::vector<int64_t> tail(G, 0);
        for (int32_t h = 0; h < G; ++h) {
            if (h == rank) {
                pp[h] = P->p_ext.get();
                px[h] = P->x_ext.get();
                mb[h] = P->mbox.get();
                continue;
            }
            void* ptr = nullptr;
            for (auto [handle, slot] : {std::pair{&exs[h].p, 0}, std::pair{&exs[h].x, 1}, std::pair{&exs[h].mb, 2}}) {
                EW_CUDA_CHECK(cudaIpcOpenMemHandle(&ptr, *handle, cudaIpcMemLazyEnablePeerAccess));
                D->ipc_mapped.push_back(ptr);
                if (slot == 0) pp[h] = static_cast<double*>(ptr);
                if (slot == 1) px[h] = static_cast<double*>(ptr);
                if (slot == 2) mb[h] = static_cast<uint64_t*>(ptr);
            }
            tail[h] = (D->bounds[h + 1] - D->bounds[h]) + before(h, rank);
        }
        peer_plan(*P, G, pp, px, mb, tail, s);
        D->peer = D->ipc = true;
        EW_CUDA_CHECK(cudaStreamSynchronize(s));
        int64_t token = rank, tokens_out[1];
        std::vector<int64_t> tokens(G);
        (void)tokens_out;
        ag(&token, tokens.data(), sizeof(token));  // every mailbox zeroed and mapped before any push
    }
    D->parts.push_back(std::move(P));
    init_overlap(*D);
    return D;
}

void dist_check_peers(const DistData& D, cudaStream_t s) {
    if (!D.peer) return;
    for (auto& P : D.parts) {
        uint64_t err = 0;
        EW_CUDA_CHECK(cudaMemcpyAsync(&err, P->mbox.get() + Mbox::err(D.nparts), sizeof(err), cudaMemcpyDeviceToHost, s));
        EW_CUDA_CHECK(cudaStreamSynchronize(s));
        if (err) {
            // the mailbox at the time of the failure: which wait was stuck
            const int32_t G = D.nparts;
            std::vector<uint64_t> mb(3 * G), ep(2);
            EW_CUDA_CHECK(cudaMemcpyAsync(mb.data(), P->mbox.get(), mb.size() * 8, cudaMemcpyDeviceToHost, s));
            EW_CUDA_CHECK(cudaMemcpyAsync(ep.data(), P->epochs.get(), 16, cudaMemcpyDeviceToHost, s));
            EW_CUDA_CHECK(cudaStreamSynchronize(s));
            std::string m = "peer transport: a peer did not answer within ~30 s (rank failure?); partition " +
                            std::to_string(P->part) + " epochs halo " + std::to_string(ep[0]) + " reduction " +
                            std::to_string(ep[1]) + "; mailbox halo/ack/red:";
            for (size_t i = 0; i < mb.size(); ++i) m += (i % G == 0 ? " |" : " ") + std::to_string(mb[i]);
            throw Error(EW_CUDA, m);
        }
    }
}

int64_t dist_owned_rows(const DistData& D) {
    int64_t n = 0;
    for (auto& P : D.parts) n += P->nloc;
    return n;
}

void dist_part_info(const DistData& D, int32_t i, int64_t* r0, int64_t* r1, int64_t* nghost, int64_t* nsend) {
    require(i >= 0 && i < static_cast<int32_t>(D.parts.size()), "no such local partition");
    const DistPart& P = *D.parts[i];
    *r0 = P.r0;
    *r1 = P.r1;
    *nghost = P.nghost;
    *nsend = static_cast<int64_t>(P.send_idx.size());
}

void dist_layout_bytes(const DistData& D, int32_t i, int64_t* slots, int64_t* bytes) {
    require(i >= 0 && i < static_cast<int32_t>(D.parts.size()), "no such local partition");
    const DistPart& P = *D.parts[i];
    *slots = *bytes = 0;
    for (const KernelData* k : {P.op_int.get(), P.op_bnd.get(), D.split ? nullptr : P.op.get()}) {
        if (!k) continue;
        *slots += k->stored_slots;
        *bytes += k->layout ? 8 * k->layout->stored_slots + layout_col_stream_bytes(*k->layout) : 12 * k->nnz;
    }
}

// y = A x over this process's owned rows (device pointers, concatenated in
// partition order).
void dist_spmv(DistData& D, const double* x, double* y, cudaStream_t s) {
    if (D.split) {  // no copies: owned x read in place, y written in place
        PartPtrs xs;
        std::vector<double*> ys;
        int64_t off = 0;
        for (auto& P : D.parts) {
            xs.push_back(x + off);
            ys.push_back(y + off);
            off += P->nloc;
        }
        spmv_exchange(D, &DistPart::x_ext, s, false, false, true, &xs, &ys);
        return;
    }
    int64_t off = 0;
    for (auto& P : D.parts) {
        if (P->nloc)
            EW_CUDA_CHECK(cudaMemcpyAsync(P->x_ext.get(), x + off, P->nloc * 8, cudaMemcpyDeviceToDevice, s));
        off += P->nloc;
    }
    spmv_exchange(D, &DistPart::x_ext, s, false, false);
    off = 0;
    for (auto& P : D.parts) {
        if (P->nloc) EW_CUDA_CHECK(cudaMemcpyAsync(y + off, P->q.get(), P->nloc * 8, cudaMemcpyDeviceToDevice, s));
        off += P->nloc;
    }
}

namespace {

// One CG iteration k (cg.cpp:69-101) of every local partition on stream t;
// k only selects the launch pattern (refresh), the kernels count iterations
// on the device.
void dist_iteration(DistData& D, const ew_cg_config& cfg, int jacobi, int64_t k, cudaStream_t t) {
    spmv_exchange(D, &DistPart::p_ext, t, true, true);
    reduce_finalize(D, cg::kPq, cfg, t);
    const bool refresh = cfg.recompute_interval > 0 && k % cfg.recompute_interval == 0;
    for (int mode : {refresh ? 1 : 0, refresh ? 2 : -1}) {
        if (mode < 0) break;
        if (mode == 2) spmv_exchange(D, &DistPart::x_ext, t, true, false);
        for (auto& P : D.parts) {
            cg::update_kernel<true><<<cg::resident_grid(cg::update_kernel<true>, cg::kRedBlock, P->nloc),
                                      cg::kRedBlock, 0, t>>>(
                mode, P->x_ext.get(), P->r.get(), P->p_ext.get(), P->q.get(), P->b.get(), P->diag.get(), P->nloc,
                jacobi, cfg.rel_tolerance, cfg.divergence_limit, P->partials.get(), P->st.get(), P->hist.get());
            launched("cg::update_kernel<dist>");
        }
    }
    reduce_finalize(D, cg::kUpdate, cfg, t);
    for (auto& P : D.parts) {
        cg::p_kernel<<<cg::resident_grid(cg::p_kernel, 256, P->nloc), 256, 0, t>>>(
            P->p_ext.get(), P->r.get(), P->diag.get(), P->nloc, jacobi, P->st.get());
        launched("cg::p_kernel");
    }
}

}  // namespace

// Everything a solve with this configuration allocates or captures: the
// working vectors, pinned polling slots and (device transports) the CUDA
// graph of one refresh block. Kept on the operator; a later solve with the
// same configuration does no allocation (cudaFree / cudaMallocHost can wait
// for the whole device, which must not happen while peers spin on this
// partition: ew_mgpu runs this for every partition before any solve starts).
void dist_cg_setup(DistData& D, const ew_cg_config& cfg, cudaStream_t s) {
    const int jacobi = cfg.jacobi ? 1 : 0;
    for (auto& P : D.parts) {
        const int64_t n = P->nloc;
        P->r.alloc(n);
        P->b.alloc(n);
        P->diag.alloc(jacobi ? n : 0);
        P->hist.alloc(cfg.max_iterations + 1);
        const int64_t spmv_blocks = (n + 255) / 256;
        P->partials.alloc(std::max<size_t>(2 * cg::kRedGridMax, cg::dot_partials(spmv_blocks)));
        P->tickets.alloc(std::max<size_t>(1, cg::dot_tickets(spmv_blocks)));
        P->st.alloc(1);
    }
    if (!D.hst) EW_CUDA_CHECK(cudaMallocHost(&D.hst, 2 * sizeof(cg::State)));
    for (auto& e : D.poll_ev)
        if (!e) EW_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    if (D.use_nccl || cfg.max_iterations <= 0) return;
    // device transports: one CUDA graph of a refresh block, replayed (the
    // comm stream joins the capture through its events)
    const int64_t interval = cfg.recompute_interval;
    const int64_t B = interval > 0 ? interval : 32;
    const int64_t hsize = static_cast<int64_t>(D.parts[0]->hist.size());
    const bool same = D.exec && D.g_tol == cfg.rel_tolerance && D.g_div == cfg.divergence_limit &&
                      D.g_interval == interval && D.g_jacobi == jacobi && D.g_hist == hsize;
    if (same) return;
    if (D.exec) cudaGraphExecDestroy(D.exec);
    D.exec = nullptr;
    if (!D.cap) EW_CUDA_CHECK(cudaStreamCreateWithFlags(&D.cap, cudaStreamNonBlocking));
    const int64_t before = g_launches.load();
    cudaGraph_t graph = nullptr;
    EW_CUDA_CHECK(cudaStreamBeginCapture(D.cap, cudaStreamCaptureModeThreadLocal));
    try {
        for (int64_t k = 1; k <= B; ++k) dist_iteration(D, cfg, jacobi, k, D.cap);
    } catch (...) {
        cudaStreamEndCapture(D.cap, &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
    }
    EW_CUDA_CHECK(cudaStreamEndCapture(D.cap, &graph));
    const cudaError_t e = cudaGraphInstantiate(&D.exec, graph, 0);
    cudaGraphDestroy(graph);
    EW_CUDA_CHECK(e);
    D.per_block = g_launches.load() - before;
    g_launches.fetch_sub(D.per_block, std::memory_order_relaxed);  // counted per replay
    D.g_tol = cfg.rel_tolerance, D.g_div = cfg.divergence_limit, D.g_interval = interval;
    D.g_jacobi = jacobi, D.g_hist = hsize;
    EW_CUDA_CHECK(cudaStreamSynchronize(s));
}

CgOutputs dist_cg(DistData& D, const double* b, const double* diag, const ew_cg_config& cfg, double* x,
                  cudaStream_t s) {
    require(cfg.rel_tolerance > 0.0, "cg: tolerance must be positive");
    require(cfg.max_iterations >= 0, "cg: max_iterations must be >= 0");
    const int jacobi = cfg.jacobi ? 1 : 0;
    if (jacobi) require(diag != nullptr, "cg: jacobi preconditioner needs the diagonal");
    dist_cg_setup(D, cfg, s);
    int64_t off = 0;
    for (auto& P : D.parts) {
        const int64_t n = P->nloc, ne = P->nloc + P->nghost;
        EW_CUDA_CHECK(cudaMemsetAsync(P->tickets.get(), 0, P->tickets.bytes(), s));
        EW_CUDA_CHECK(cudaMemsetAsync(P->st.get(), 0, sizeof(cg::State), s));
        const long long max_it = cfg.max_iterations;
        EW_CUDA_CHECK(cudaMemcpyAsync(&P->st.get()->max_it, &max_it, sizeof(max_it), cudaMemcpyHostToDevice, s));
        if (ne) {
            EW_CUDA_CHECK(cudaMemsetAsync(P->x_ext.get(), 0, ne * 8, s));
            EW_CUDA_CHECK(cudaMemsetAsync(P->p_ext.get(), 0, ne * 8, s));
        }
        if (n) {
            EW_CUDA_CHECK(cudaMemcpyAsync(P->b.get(), b + off, n * 8, cudaMemcpyDeviceToDevice, s));
            if (jacobi) EW_CUDA_CHECK(cudaMemcpyAsync(P->diag.get(), diag + off, n * 8, cudaMemcpyDeviceToDevice, s));
        }
        off += n;
    }
    // ||b||, then the global OR of the local pre-check flags (cg.cpp:28-33)
    for (auto& P : D.parts) {
        cg::init_kernel<true><<<cg::red_grid(P->nloc), cg::kRedBlock, 0, s>>>(P->b.get(), P->diag.get(), P->nloc,
                                                                              jacobi, P->partials.get(), P->st.get());
        launched("cg::init_kernel<dist>");
    }
    reduce_finalize(D, cg::kBnorm, cfg, s);
    cg::State* hst = static_cast<cg::State*>(D.hst);
    std::vector<cg::State> hs(D.parts.size());
    for (size_t i = 0; i < D.parts.size(); ++i) {
        EW_CUDA_CHECK(cudaMemcpyAsync(&hst[0], D.parts[i]->st.get(), sizeof(cg::State), cudaMemcpyDeviceToHost, s));
        EW_CUDA_CHECK(cudaStreamSynchronize(s));
        hs[i] = hst[0];
    }
    double flags[2] = {0.0, 0.0};
    for (auto& h : hs) {
        if (h.status == cg::kBadRhs) flags[0] = 1.0;
        if (h.flags & 2) flags[1] = 1.0;
    }
    if (D.use_nccl || D.ipc) {  // share the flags: all ranks take the same branch
        DistPart& P = *D.parts[0];
        EW_CUDA_CHECK(cudaMemcpyAsync(P.st.get()->loc, flags, 16, cudaMemcpyHostToDevice, s));
        allgather(D, s);
        std::vector<double> all(2 * static_cast<size_t>(D.nparts));
        EW_CUDA_CHECK(cudaMemcpyAsync(all.data(), P.gathered.get(), all.size() * 8, cudaMemcpyDeviceToHost, s));
        EW_CUDA_CHECK(cudaStreamSynchronize(s));
        for (int32_t g = 0; g < D.nparts; ++g) {
            flags[0] = std::max(flags[0], all[2 * g]);
            flags[1] = std::max(flags[1], all[2 * g + 1]);
        }
    }
    if (flags[0] != 0.0) throw Error(EW_CG_DIVERGENCE, "cg: non-finite right-hand side");
    require(flags[1] == 0.0, "cg: zero diagonal entry under jacobi");
    CgOutputs out;
    if (hs[0].bnorm == 0.0) {
        out.res.converged = 1;
        out.res.history_len = 1;
        out.history.assign(1, 0.0);
        cudaMemsetAsync(x, 0, dist_owned_rows(D) * 8, s);
        EW_CUDA_CHECK(cudaStreamSynchronize(s));
        return out;
    }
    // r = b - A x0 (x0 = 0; the operator still runs, cg.cpp:52-57)
    spmv_exchange(D, &DistPart::x_ext, s, false, false, /*exchange=*/false);  // x0 = 0 everywhere
    for (auto& P : D.parts) {
        cg::start_kernel<true><<<cg::red_grid(P->nloc), cg::kRedBlock, 0, s>>>(
            P->b.get(), P->diag.get(), P->q.get(), P->r.get(), P->p_ext.get(), P->nloc, jacobi, cfg.rel_tolerance,
            P->partials.get(), P->st.get(), P->hist.get());
        launched("cg::start_kernel<dist>");
    }
    reduce_finalize(D, cg::kStart, cfg, s);

    DistPart& P0 = *D.parts[0];
    cudaEvent_t* ev = D.poll_ev;
    // every rank launches the same blocks and stops on the same polled
    // state (identical decisions everywhere), so the exchanges pair up
    int j = 0;
    auto poll = [&]() -> bool {
        const int slot = j & 1;
        EW_CUDA_CHECK(cudaMemcpyAsync(&hst[slot], P0.st.get(), sizeof(cg::State), cudaMemcpyDeviceToHost, s));
        EW_CUDA_CHECK(cudaEventRecord(ev[slot], s));
        bool stop = false;
        if (j > 0) {
            EW_CUDA_CHECK(cudaEventSynchronize(ev[slot ^ 1]));
            stop = hst[slot ^ 1].done != 0;
        }
        ++j;
        return stop;
    };
    const int64_t interval = cfg.recompute_interval;
    if (!D.use_nccl && cfg.max_iterations > 0) {
        const int64_t B = interval > 0 ? interval : 32;
        const int64_t blocks = (cfg.max_iterations + B - 1) / B;
        for (int64_t blk = 0; blk < blocks; ++blk) {
            EW_CUDA_CHECK(cudaGraphLaunch(D.exec, s));
            g_launches.fetch_add(D.per_block, std::memory_order_relaxed);
            if (poll()) break;
        }
    } else {
        int64_t it = 1;
        int batch = 8;
        while (it <= cfg.max_iterations) {
            const int64_t last = std::min<int64_t>(cfg.max_iterations, it + batch - 1);
            for (; it <= last; ++it) dist_iteration(D, cfg, jacobi, it, s);
            if (poll()) break;
            batch = std::min(batch * 2, 64);
        }
    }
    EW_CUDA_CHECK(cudaMemcpyAsync(&hst[0], P0.st.get(), sizeof(cg::State), cudaMemcpyDeviceToHost, s));
    EW_CUDA_CHECK(cudaStreamSynchronize(s));
    const cg::State h = hst[0];
    off = 0;
    for (auto& P : D.parts) {
        if (P->nloc) EW_CUDA_CHECK(cudaMemcpyAsync(x + off, P->x_ext.get(), P->nloc * 8, cudaMemcpyDeviceToDevice, s));
        off += P->nloc;
    }
    EW_CUDA_CHECK(cudaStreamSynchronize(s));
    dist_check_peers(D, s);
    return cg_outputs(h.status, h.iterations, cfg, P0.hist.get());
}

// ---- single process, several GPUs (SURVEY.md §8(b) ew_mgpu_cg_solve) --------
// One DistData per partition, exactly as one rank of the CUDA-IPC transport
// (the same push / mailbox / publish kernels, one partition per operator),
// but the peers are this process's other partitions on other devices (or
// the same one): their ghost buffers and mailboxes are plain device pointers
// reached through peer access, and each partition's solve runs on its own
// host thread and stream.
struct MgpuData {
    int32_t G = 0;
    int64_t n = 0;
    std::vector<int> dev;
    std::vector<int64_t> bounds;
    std::vector<std::shared_ptr<DistData>> parts;
    std::vector<cudaStream_t> streams;
    ~MgpuData() {
        int prev = 0;
        cudaGetDevice(&prev);
        // each block's buffers, graph and streams with its own device current
        for (size_t g = 0; g < parts.size(); ++g) {
            cudaSetDevice(dev[g]);
            parts[g].reset();
        }
        for (size_t g = 0; g < streams.size(); ++g) {
            cudaSetDevice(dev[g]);
            cudaStreamDestroy(streams[g]);
        }
        cudaSetDevice(prev);
    }
};

namespace {

struct DeviceGuard {
    int prev = 0;
    DeviceGuard() { cudaGetDevice(&prev); }
    ~DeviceGuard() { cudaSetDevice(prev); }
};

// Runs fn(g) for every partition on its own thread (device set), rethrowing
// the first failure.
template <typename Fn>
void on_every_part(MgpuData& M, Fn&& fn) {
    std::vector<std::exception_ptr> err(M.G);
    std::vector<std::thread> th;
    for (int32_t g = 0; g < M.G; ++g)
        th.emplace_back([&, g] {
            try {
                EW_CUDA_CHECK(cudaSetDevice(M.dev[g]));
                fn(g);
            } catch (...) {
                err[g] = std::current_exception();
            }
        });
    for (auto& t : th) t.join();
    for (auto& e : err)
        if (e) std::rethrow_exception(e);
}

}  // namespace

std::shared_ptr<MgpuData> mgpu_create(int64_t n, const int64_t* ro, const int64_t* ci, const double* v,
                                      int32_t G, const int32_t* devices, const std::string& kid,
                                      const ew_warp_config& cfg, const ew_kernel_options& opts) {
    require(G >= 1, "mgpu: need at least one partition");
    require(kid == "k1" || kid == "k2" || kid == "csr_ref",
            "partitioned kernels: k1, k2 or csr_ref (the local matrix has ghost columns)");
    int ndev = 0;
    EW_CUDA_CHECK(cudaGetDeviceCount(&ndev));
    DeviceGuard guard;
    auto M = std::make_shared<MgpuData>();
    M->G = G;
    M->n = n;
    for (int32_t g = 0; g < G; ++g) {
        const int d = devices ? devices[g] : g;
        require(d >= 0 && d < ndev, "mgpu: device " + std::to_string(d) + " does not exist");
        M->dev.push_back(d);
    }
    M->bounds = partition_rows(ro, n, G);
    // every partition's ghosts from the global CSR; peer access between the devices
    std::vector<std::vector<int64_t>> ghosts(G);
    for (int32_t h = 0; h < G; ++h) ghosts[h] = ghost_list(ro + M->bounds[h], ci, M->bounds[h], M->bounds[h + 1]);
    for (int32_t a = 0; a < G; ++a)
        for (int32_t b = 0; b < G; ++b) {
            if (M->dev[a] == M->dev[b]) continue;
            int ok = 0;
            EW_CUDA_CHECK(cudaDeviceCanAccessPeer(&ok, M->dev[a], M->dev[b]));
            require(ok, "mgpu: device " + std::to_string(M->dev[a]) + " cannot access device " +
                            std::to_string(M->dev[b]) + " (no peer access)");
            EW_CUDA_CHECK(cudaSetDevice(M->dev[a]));
            const cudaError_t e = cudaDeviceEnablePeerAccess(M->dev[b], 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) (void)cudaGetLastError();
            else EW_CUDA_CHECK(e);
        }
    for (int32_t g = 0; g < G; ++g) {
        EW_CUDA_CHECK(cudaSetDevice(M->dev[g]));
        cudaStream_t s = nullptr;
        EW_CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        M->streams.push_back(s);
        std::vector<std::vector<int64_t>> needs(G);
        for (int32_t h = 0; h < G; ++h) {
            if (h == g) continue;
            for (int64_t c : ghosts[h])
                if (c >= M->bounds[g] && c < M->bounds[g + 1]) needs[h].push_back(c);
        }
        auto D = std::make_shared<DistData>();
        D->nparts = G;
        D->first = g;
        D->nlocal = 1;
        D->kernel_id = kid;
        D->bounds = M->bounds;
        auto P = std::make_unique<DistPart>();
        build_part(*P, g, G, D->bounds, ro + M->bounds[g], ci, v, ghosts[g], needs, kid, cfg, opts, s);
        if (G > 1) alloc_mailbox(*P, G, s);
        D->parts.push_back(std::move(P));
        M->parts.push_back(D);
    }
    if (G > 1) {
        std::vector<double*> pp(G), px(G);
        std::vector<uint64_t*> mb(G);
        for (int32_t h = 0; h < G; ++h) {
            DistPart& H = *M->parts[h]->parts[0];
            pp[h] = H.p_ext.get();
            px[h] = H.x_ext.get();
            mb[h] = H.mbox.get();
        }
        for (int32_t g = 0; g < G; ++g) {
            EW_CUDA_CHECK(cudaSetDevice(M->dev[g]));
            DistPart& P = *M->parts[g]->parts[0];
            std::vector<int64_t> tail(G, 0);
            for (int32_t h = 0; h < G; ++h) {
                if (h == g) continue;
                const DistPart& H = *M->parts[h]->parts[0];
                tail[h] = H.nloc + H.recv_off[g];
            }
            peer_plan(P, G, pp, px, mb, tail, M->streams[g]);
            M->parts[g]->peer = M->parts[g]->ipc = true;  // one partition per operator, peers elsewhere
        }
    }
    for (int32_t g = 0; g < G; ++g) {
        EW_CUDA_CHECK(cudaSetDevice(M->dev[g]));
        init_overlap(*M->parts[g]);
        EW_CUDA_CHECK(cudaStreamSynchronize(M->streams[g]));
    }
    return M;
}

int64_t mgpu_rows(const MgpuData& M) { return M.n; }

// y = A x, host vectors of n entries.
void mgpu_spmv(MgpuData& M, const double* x, double* y) {
    on_every_part(M, [&](int32_t g) {
        const int64_t r0 = M.bounds[g], nl = M.bounds[g + 1] - r0;
        const cudaStream_t s = M.streams[g];
        Scratch<double> xd(nl, s), yd(nl, s);
        if (nl) EW_CUDA_CHECK(cudaMemcpyAsync(xd.get(), x + r0, nl * 8, cudaMemcpyHostToDevice, s));
        dist_spmv(*M.parts[g], xd.get(), yd.get(), s);
        if (nl) EW_CUDA_CHECK(cudaMemcpyAsync(y + r0, yd.get(), nl * 8, cudaMemcpyDeviceToHost, s));
        EW_CUDA_CHECK(cudaStreamSynchronize(s));
        dist_check_peers(*M.parts[g], s);
    });
}

// cg_solve over all partitions (host b, diag, x of n entries); every
// partition takes the same decisions, partition 0 reports.
CgOutputs mgpu_cg(MgpuData& M, const double* b, const double* diag, const ew_cg_config& cfg, double* x) {
    const bool jac = cfg.jacobi != 0;
    require(!jac || diag != nullptr, "cg: jacobi preconditioner needs the diagonal");
    std::vector<CgOutputs> out(M.G);
    // allocations and graph capture of every partition first: none of them
    // may wait for the device while another partition's kernels spin
    on_every_part(M, [&](int32_t g) { dist_cg_setup(*M.parts[g], cfg, M.streams[g]); });
    on_every_part(M, [&](int32_t g) {
        const int64_t r0 = M.bounds[g], nl = M.bounds[g + 1] - r0;
        const cudaStream_t s = M.streams[g];
        Scratch<double> bd(nl, s), dd(jac ? nl : 0, s), xd(nl, s);
        if (nl) {
            EW_CUDA_CHECK(cudaMemcpyAsync(bd.get(), b + r0, nl * 8, cudaMemcpyHostToDevice, s));
            if (jac) EW_CUDA_CHECK(cudaMemcpyAsync(dd.get(), diag + r0, nl * 8, cudaMemcpyHostToDevice, s));
        }
        out[g] = dist_cg(*M.parts[g], bd.get(), jac ? dd.get() : nullptr, cfg, xd.get(), s);
        if (nl) EW_CUDA_CHECK(cudaMemcpyAsync(x + r0, xd.get(), nl * 8, cudaMemcpyDeviceToHost, s));
        EW_CUDA_CHECK(cudaStreamSynchronize(s));
    });
    return out[0];
}

void nccl_unique_id(void* out) {
    ncclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, sizeof(id));
}

const void* kernel_anchor_dist() { return reinterpret_cast<const void*>(&pack_kernel); }

}  // namespace ew

// PCIe probe for the host-buffer apply pipeline (ew_kernel.cu): moves one
// config-2 call's bytes (x up, y down: 15.8 MB each) four ways and times
// them with CUDA events -- copy engines both ways; an SM kernel writing y
// into mapped pinned memory while a copy engine uploads x; an SM kernel
// reading x from mapped memory while a copy engine downloads y; SM kernels
// both ways. Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
// tools/pcie_probe.cu -o tools/pcie_probe
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                  \
    do {                                                                       \
        cudaError_t e = (x);                                                   \
        if (e != cudaSuccess) {                                                \
            std::printf("%s: %s\n", #x, cudaGetErrorString(e));                \
            std::exit(1);                                                      \
        }                                                                      \
    } while (0)

__global__ void zc_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

// HBM load beside the copies: streams `n` 16-byte words (reads) per call.
__global__ void hog(const uint4* __restrict__ src, size_t n, unsigned* sink) {
    unsigned acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const uint4 v = __ldcs(src + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u) *sink = acc;
}

int main(int argc, char** argv) {
    const size_t bytes = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 15804072;
    const int ctas = argc > 2 ? std::atoi(argv[2]) : 64;
    const size_t n16 = bytes / 16;
    void *hx, *hy, *dx, *dy, *hx_d, *hy_d;
    CK(cudaHostAlloc(&hx, bytes, cudaHostAllocMapped));
    CK(cudaHostAlloc(&hy, bytes, cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer(&hx_d, hx, 0));
    CK(cudaHostGetDevicePointer(&hy_d, hy, 0));
    CK(cudaMalloc(&dx, bytes));
    CK(cudaMalloc(&dy, bytes));
    cudaStream_t a, b;
    CK(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking));
    cudaEvent_t e0, ea, eb, ej;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&ea));
    CK(cudaEventCreate(&eb));
    CK(cudaEventCreate(&ej));
    const size_t hog_bytes = argc > 3 ? std::strtoull(argv[3], nullptr, 10) : 0;
    const int hog_ctas = argc > 4 ? std::atoi(argv[4]) : 148 * 8;
    const int chunks = argc > 5 ? std::atoi(argv[5]) : 1;  // copy-engine copies per direction
    const int ustreams = argc > 6 ? std::atoi(argv[6]) : 1;  // upload chunk k on stream k % ustreams
    cudaStream_t us[8];
    cudaEvent_t ue[8];
    for (int i = 0; i < 8; ++i) {
        CK(cudaStreamCreateWithFlags(&us[i], cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&ue[i], cudaEventDisableTiming));
    }
    void* hbuf = nullptr;
    unsigned* sink = nullptr;
    cudaStream_t c;
    CK(cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking));
    if (hog_bytes) {
        CK(cudaMalloc(&hbuf, hog_bytes));
        CK(cudaMemset(hbuf, 1, hog_bytes));
        CK(cudaMalloc(&sink, 4));
    }
    const char* names[] = {"CE up | CE down", "CE up | SM down", "SM up | CE down", "SM up | SM down",
                           "CE up alone", "CE down alone", "SM up alone", "SM down alone", "hog alone"};
    for (int mode = 0; mode < 9; ++mode) {
        if (mode == 8 && !hog_bytes) break;
        if (hog_bytes && mode != 0 && mode != 4 && mode != 5 && mode != 8) continue;
        float best = 1e9f, tot = 0.0f;
        const int reps = 20;
        for (int r = 0; r < reps + 3; ++r) {
            CK(cudaEventRecord(e0, a));
            CK(cudaStreamWaitEvent(b, e0, 0));
            if (hog_bytes) {
                CK(cudaStreamWaitEvent(c, e0, 0));
                hog<<<hog_ctas, 256, 0, c>>>((const uint4*)hbuf, hog_bytes / 16, sink);
            }
            const bool up = mode != 5 && mode != 7 && mode != 8, down = mode != 4 && mode != 6 && mode != 8;
            const bool sm_up = mode == 2 || mode == 3 || mode == 6, sm_down = mode == 1 || mode == 3 || mode == 7;
            if (up) {
                if (sm_up) zc_copy<<<ctas, 256, 0, a>>>((const uint4*)hx_d, (uint4*)dx, n16);
                else {
                    for (int i = 1; i < ustreams; ++i) CK(cudaStreamWaitEvent(us[i], e0, 0));
                    for (int k = 0; k < chunks; ++k) {
                        const size_t o = bytes * k / chunks / 16 * 16, end = bytes * (k + 1) / chunks / 16 * 16;
                        cudaStream_t u = k % ustreams == 0 ? a : us[k % ustreams];
                        CK(cudaMemcpyAsync((char*)dx + o, (char*)hx + o, end - o, cudaMemcpyHostToDevice, u));
                    }
                    for (int i = 1; i < ustreams; ++i) {
                        CK(cudaEventRecord(ue[i], us[i]));
                        CK(cudaStreamWaitEvent(a, ue[i], 0));
                    }
                }
            }
            if (down) {
                if (sm_down) zc_copy<<<ctas, 256, 0, b>>>((const uint4*)dy, (uint4*)hy_d, n16);
                else
                    for (int k = 0; k < chunks; ++k) {
                        const size_t o = bytes * k / chunks / 16 * 16, end = bytes * (k + 1) / chunks / 16 * 16;
                        CK(cudaMemcpyAsync((char*)hy + o, (char*)dy + o, end - o, cudaMemcpyDeviceToHost, b));
                    }
            }
            CK(cudaEventRecord(eb, b));
            CK(cudaStreamWaitEvent(a, eb, 0));
            if (hog_bytes) {
                CK(cudaEventRecord(ea, c));
                CK(cudaStreamWaitEvent(a, ea, 0));
            }
            CK(cudaEventRecord(ej, a));
            CK(cudaEventSynchronize(ej));
            float ms = 0.0f;
            CK(cudaEventElapsedTime(&ms, e0, ej));
            if (r >= 3) {
                tot += ms;
                if (ms < best) best = ms;
            }
        }
        std::printf("%-18s bytes %zu chunks %d/%d ctas %3d hog %zu/%d: best %.4f ms, mean %.4f ms\n", names[mode], bytes,
                    chunks, ustreams, ctas, hog_bytes, hog_ctas, best, tot / reps);
    }
    return 0;
}
